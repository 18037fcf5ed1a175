// sweep_onesweep.cu — developer tool: time one LSD node-key pass of k_onesweep under several
// (THREADS, ITEMS, look-back window, min blocks/SM, BINS) configurations on a config-5-like key
// set (Kuhn n^3 tets, b = 25 node bits), and check every variant writes the same output.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1604_04689_b200/csrc \
//        tools/sweep_onesweep.cu -o tools/sweep_onesweep && ./tools/sweep_onesweep [n]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "kernels.cuh"

using namespace mn;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__global__ void gen_kuhn(int n, int32_t* conn) {
  const int64_t ncell = (int64_t)n * n * n;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ci = c % n, cj = (c / n) % n, ck = c / ((int64_t)n * n);
    const int64_t w = n + 1;
    const int64_t base = ci + w * (cj + w * ck);
    const int64_t step[3] = {1, w, w * w};
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int p = 0; p < 6; ++p) {
      int32_t* t = conn + (c * 6 + p) * 4;
      t[0] = (int32_t)base;
      t[1] = (int32_t)(base + step[perms[p][0]]);
      t[2] = (int32_t)(base + step[perms[p][0]] + step[perms[p][1]]);
      t[3] = (int32_t)(base + 1 + w + w * w);
    }
  }
}

__global__ void hist_digit(const uint64_t* keys, int64_t n, int shift, uint32_t mask, unsigned long long* h) {
  __shared__ unsigned int sh[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&sh[(keys[i] >> shift) & mask], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) if (sh[i]) atomicAdd(h + i, (unsigned long long)sh[i]);
}

__global__ void checksum(const uint64_t* k, int64_t n, unsigned long long* out) {
  unsigned long long acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += (k[i] * 0x9E3779B97F4A7C15ull) ^ (unsigned long long)i;
  atomicAdd(out, acc);
}

struct Ctx {
  uint64_t *A, *B;
  int64_t n;
  uint64_t* status;
  uint32_t* ticket;
  uint64_t* bases;
  unsigned long long* err;
  size_t status_bytes;
};

template <int BINS, int THREADS, int ITEMS, int W, int MINB>
void run_variant(Ctx& c, int shift, int width, const char* label, unsigned long long ref_sum) {
  using Sm = OnesweepSmem<THREADS, ITEMS, BINS>;
  constexpr int TILE = THREADS * ITEMS;
  const int64_t tiles = (c.n + TILE - 1) / TILE;
  const size_t smem = ((sizeof(Sm) + 15) & ~size_t(15)) + (size_t)TILE * 8;
  auto kern = k_onesweep<uint64_t, 0, 0, false, false, BINS, THREADS, ITEMS, W, MINB>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, smem));
  // bases for this digit
  std::vector<unsigned long long> h(512, 0);
  unsigned long long* dh;
  CK(cudaMalloc(&dh, 512 * 8));
  CK(cudaMemset(dh, 0, 512 * 8));
  hist_digit<<<148 * 8, 256>>>(c.A, c.n, shift, (1u << width) - 1, dh);
  CK(cudaMemcpy(h.data(), dh, 512 * 8, cudaMemcpyDeviceToHost));
  std::vector<uint64_t> b(BINS, 0);
  uint64_t run = 0;
  for (int i = 0; i < BINS; ++i) { b[i] = run; run += h[i]; }
  CK(cudaMemcpy(c.bases, b.data(), BINS * 8, cudaMemcpyHostToDevice));
  PassArgs pa{};
  pa.keys_in = c.A; pa.keys_out = c.B; pa.n = c.n;
  pa.pd.shift = shift; pa.pd.mask = (1u << width) - 1; pa.pd.div = 1;
  pa.bases = c.bases; pa.status = c.status; pa.ticket = c.ticket; pa.err = c.err;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int rep = 0; rep < 6; ++rep) {
    CK(cudaMemset(c.status, 0, (size_t)tiles * BINS * 8));
    CK(cudaMemset(c.ticket, 0, 4));
    pa.epoch = 1;
    cudaEventRecord(e0);
    kern<<<(unsigned)tiles, THREADS, smem>>>(pa);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep) ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  const float ms = ts[ts.size() / 2];
  CK(cudaMemset(dh, 0, 8));
  checksum<<<148 * 8, 256>>>(c.B, c.n, dh);
  unsigned long long sum = 0;
  CK(cudaMemcpy(&sum, dh, 8, cudaMemcpyDeviceToHost));
  cudaFree(dh);
  printf("%-34s bins=%3d thr=%3d items=%2d W=%2d minB=%d occ=%d tiles=%8lld smem=%6zu : %8.3f ms  %7.1f GB/s  %s\n",
         label, BINS, THREADS, ITEMS, W, MINB, occ, (long long)tiles, smem, ms, 16.0 * c.n / (ms * 1e-3) / 1e9,
         ref_sum == 0 ? "" : (sum == ref_sum ? "ok" : "MISMATCH"));
  fflush(stdout);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 256;
  const int64_t M = 6LL * n * n * n;
  const int64_t N = (int64_t)(n + 1) * (n + 1) * (n + 1);
  int b = 0; { uint64_t x = N - 1; while (x) { ++b; x >>= 1; } }
  const int64_t P = 12 * M;
  printf("Kuhn %d^3: M=%lld N=%lld b=%d node pairs=%lld (%.2f GB keys)\n", n, (long long)M, (long long)N, b,
         (long long)P, P * 8.0 / 1e9);
  int32_t* conn;
  Ctx c{};
  c.n = P;
  CK(cudaMalloc(&conn, M * 16));
  CK(cudaMalloc(&c.A, P * 8));
  CK(cudaMalloc(&c.B, P * 8));
  const int64_t max_tiles = P / 2048 + 2;
  CK(cudaMalloc(&c.status, max_tiles * 512 * 8));
  CK(cudaMalloc(&c.ticket, 64));
  CK(cudaMalloc(&c.bases, 512 * 8));
  CK(cudaMalloc(&c.err, 8));
  CK(cudaMemset(c.err, 0xFF, 8));
  gen_kuhn<<<148 * 8, 256>>>(n, conn);
  CK(cudaGetLastError());
  // Keys as the path produces them after pass 0: emit (slot order) — then one pass on the lowest
  // 9 bits (like pass 0) so the input of the timed pass has the real pass-1 structure.
  k_emit_node<MN_TET4, uint64_t><<<148 * 16, 256>>>(conn, P, b, c.A, c.err);
  CK(cudaDeviceSynchronize());
  const int w0 = (b + 2) / 3;   // 9,8,8 for b = 25
  {
    // pre-pass: sort A on digit 0 into B, swap
    Ctx d = c;
    run_variant<512, 256, 16, 4, 3>(d, 0, w0, "prepass (digit 0)", 0);
    std::swap(c.A, c.B);
  }
  const int s1 = w0, wd1 = (b - w0 + 1) / 2;   // timed digit 1 of the v part
  unsigned long long ref = 0;
  {
    // reference output of the timed pass
    run_variant<512, 256, 16, 1, 3>(c, s1, wd1, "ref W=1 (serial walk)", 0);
    unsigned long long* dh; CK(cudaMalloc(&dh, 8)); CK(cudaMemset(dh, 0, 8));
    checksum<<<148 * 8, 256>>>(c.B, c.n, dh);
    CK(cudaMemcpy(&ref, dh, 8, cudaMemcpyDeviceToHost));
    cudaFree(dh);
  }
  run_variant<512, 256, 16, 2, 3>(c, s1, wd1, "W=2", ref);
  run_variant<512, 256, 16, 4, 3>(c, s1, wd1, "W=4", ref);
  run_variant<512, 256, 16, 8, 3>(c, s1, wd1, "W=8", ref);
  run_variant<512, 256, 16, 16, 2>(c, s1, wd1, "W=16", ref);
  run_variant<512, 256, 16, 4, 2>(c, s1, wd1, "W=4 minB2", ref);
  run_variant<512, 256, 24, 4, 2>(c, s1, wd1, "items24", ref);
  run_variant<512, 256, 32, 4, 2>(c, s1, wd1, "items32", ref);
  run_variant<512, 512, 16, 4, 2>(c, s1, wd1, "thr512", ref);
  run_variant<512, 512, 16, 8, 2>(c, s1, wd1, "thr512 W8", ref);
  run_variant<512, 512, 16, 4, 1>(c, s1, wd1, "thr512 minB1", ref);
  run_variant<512, 512, 24, 4, 1>(c, s1, wd1, "thr512 items24", ref);
  // 8-bit digit at the same shift (a different, 256-bin pass: timing only)
  run_variant<256, 256, 16, 1, 3>(c, s1, 8, "8-bit W=1", 0);
  run_variant<256, 256, 16, 4, 3>(c, s1, 8, "8-bit W=4", 0);
  run_variant<256, 256, 16, 8, 3>(c, s1, 8, "8-bit W=8", 0);
  run_variant<256, 256, 24, 4, 2>(c, s1, 8, "8-bit items24", 0);
  // plain copy for scale
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    std::vector<float> ts;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      CK(cudaMemcpyAsync(c.B, c.A, P * 8, cudaMemcpyDeviceToDevice));
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    printf("cudaMemcpy D2D same bytes: %.3f ms %.1f GB/s\n", ts[2], 16.0 * P / (ts[2] * 1e-3) / 1e9);
  }
  return 0;
}
