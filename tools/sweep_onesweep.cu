// sweep_onesweep.cu — developer tool: time single k_onesweep passes under different kernel
// configurations (ranking method, tile shape, look-back window, occupancy) on element-pair keys
// as the pipeline produces them (u32 node key + u32 element payload), for a coherent mesh (Kuhn
// tets, natural numbering) and for randomly numbered nodes; each variant's output is checked
// against the first variant of its group.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1604_04689_b200/csrc \
//        tools/sweep_onesweep.cu -o tools/sweep_onesweep && ./tools/sweep_onesweep [n]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

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

// random relabelling inside [0, 2^b): an odd multiplier is a bijection modulo 2^b
__global__ void scramble(int32_t* conn, int64_t n, int b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    conn[i] = (int32_t)(((uint32_t)conn[i] * 2654435761u + 12345u) & ((1u << b) - 1u));
}

template <typename KeyT>
__global__ void hist_digit(const KeyT* keys, int64_t n, int shift, uint32_t mask, unsigned long long* h) {
  __shared__ unsigned int sh[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&sh[(keys[i] >> shift) & mask], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) if (sh[i]) atomicAdd(h + i, (unsigned long long)sh[i]);
}

template <typename KeyT>
__global__ void checksum(const KeyT* k, const uint32_t* v, int64_t n, unsigned long long* out) {
  unsigned long long acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += ((unsigned long long)k[i] * 0x9E3779B97F4A7C15ull) ^ ((unsigned long long)i << 7) ^ (v ? v[i] * 31ull : 0ull);
  atomicAdd(out, acc);
}

struct Bufs {
  void *kA, *kB;
  uint32_t *vA, *vB;
  int64_t n;
  uint64_t* status;
  uint32_t* ticket;
  uint64_t* bases;
  unsigned long long* err;
  const int32_t* conn;
};

template <typename KeyT, int SRC, int T, bool PAYLOAD, int BINS, int THREADS, int ITEMS, int W, int MINB, int RANK,
          bool EARLY = false>
unsigned long long run(Bufs& c, int shift, int width, const char* label, unsigned long long ref) {
  using Sm = OnesweepSmem<THREADS, ITEMS, BINS>;
  constexpr int TILE = THREADS * ITEMS;
  const int64_t tiles = (c.n + TILE - 1) / TILE;
  const size_t smem = ((sizeof(Sm) + 15) & ~size_t(15)) + (size_t)TILE * sizeof(KeyT) + ((PAYLOAD || SRC == 2) ? (size_t)TILE * 4 : 0);
  auto kern = k_onesweep<KeyT, SRC, T, PAYLOAD, false, BINS, THREADS, ITEMS, W, MINB, RANK, false, EARLY>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, smem));
  // bases of this digit: from the input keys (SRC 0) or from conn (SRC 2)
  unsigned long long* dh;
  CK(cudaMalloc(&dh, 512 * 8));
  CK(cudaMemset(dh, 0, 512 * 8));
  if (SRC == 0) hist_digit<KeyT><<<148 * 8, 256>>>((const KeyT*)c.kA, c.n, shift, (1u << width) - 1, dh);
  else hist_digit<int32_t><<<148 * 8, 256>>>(c.conn, c.n, shift, (1u << width) - 1, dh);
  std::vector<unsigned long long> h(512);
  CK(cudaMemcpy(h.data(), dh, 512 * 8, cudaMemcpyDeviceToHost));
  std::vector<uint64_t> b(BINS);
  uint64_t acc = 0;
  for (int i = 0; i < BINS; ++i) { b[i] = acc; acc += h[i]; }
  CK(cudaMemcpy(c.bases, b.data(), BINS * 8, cudaMemcpyHostToDevice));
  PassArgs pa{};
  pa.keys_in = c.kA; pa.keys_out = c.kB; pa.vals_in = c.vA; pa.vals_out = c.vB; pa.conn = c.conn; pa.n = c.n;
  pa.pd.shift = shift; pa.pd.mask = (1u << width) - 1; pa.pd.div = 1;
  pa.bases = c.bases; pa.status = c.status; pa.ticket = c.ticket; pa.err = c.err; pa.epoch = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int rep = 0; rep < 6; ++rep) {
    CK(cudaMemset(c.status, 0, (size_t)tiles * BINS * 8));
    CK(cudaMemset(c.ticket, 0, 4));
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
  checksum<KeyT><<<148 * 8, 256>>>((const KeyT*)c.kB, PAYLOAD || SRC == 2 ? c.vB : nullptr, c.n, dh);
  unsigned long long sum = 0;
  CK(cudaMemcpy(&sum, dh, 8, cudaMemcpyDeviceToHost));
  cudaFree(dh);
  const double bytes = SRC == 2 ? 12.0 * c.n : (PAYLOAD ? 16.0 : 2.0 * sizeof(KeyT)) * c.n;
  printf("%-26s bins=%3d thr=%3d items=%2d W=%d minB=%d rank=%d occ=%d : %7.3f ms %7.1f GB/s %s\n", label, BINS,
         THREADS, ITEMS, W, MINB, RANK, occ, ms, bytes / (ms * 1e-3) / 1e9, ref == 0 ? "" : (sum == ref ? "ok" : "MISMATCH"));
  fflush(stdout);
  return sum;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 256;
  const int64_t M = 6LL * n * n * n, N = (int64_t)(n + 1) * (n + 1) * (n + 1);
  int b = 0; { uint64_t x = N - 1; while (x) { ++b; x >>= 1; } }
  const int64_t P = 4 * M;
  printf("Kuhn %d^3: M=%lld N=%lld b=%d element pairs=%lld\n", n, (long long)M, (long long)N, b, (long long)P);
  int32_t* conn;
  Bufs c{};
  c.n = P;
  CK(cudaMalloc(&conn, P * 4));
  CK(cudaMalloc(&c.kA, P * 8));
  CK(cudaMalloc(&c.kB, P * 8));
  CK(cudaMalloc(&c.vA, P * 4));
  CK(cudaMalloc(&c.vB, P * 4));
  CK(cudaMalloc(&c.status, (P / 2048 + 2) * 512 * 8));
  CK(cudaMalloc(&c.ticket, 64));
  CK(cudaMalloc(&c.bases, 512 * 8));
  CK(cudaMalloc(&c.err, 8));
  CK(cudaMemset(c.err, 0xFF, 8));
  c.conn = conn;
  const int w0 = (b + 2) / 3, w1 = (b - w0 + 1) / 2;
  for (int scr = 0; scr < 1; ++scr) {
    gen_kuhn<<<148 * 8, 256>>>(n, conn);
    if (scr) scramble<<<148 * 8, 256>>>(conn, P, b);
    CK(cudaDeviceSynchronize());
    printf("---- %s node numbering ----\n", scr ? "random" : "natural (coherent)");
    // pass 0 from conn
    unsigned long long r0 = run<uint32_t, 2, MN_TET4, false, 512, 512, 16, 4, 2, 0>(c, 0, w0, "pass0 match", 0);
    run<uint32_t, 2, MN_TET4, false, 512, 512, 16, 4, 2, 0, true>(c, 0, w0, "pass0 early", r0);
    run<uint32_t, 2, MN_TET4, false, 512, 512, 16, 8, 2, 0, true>(c, 0, w0, "pass0 early W8", r0);
    // make the pass-0 output the input of the timed pass 1
    std::swap(c.kA, c.kB);
    std::swap(c.vA, c.vB);
    unsigned long long r1 = run<uint32_t, 0, 0, true, 512, 512, 16, 4, 2, 0>(c, w0, w1, "pass1 match", 0);
    run<uint32_t, 0, 0, true, 512, 512, 16, 4, 2, 0, true>(c, w0, w1, "pass1 early", r1);
    run<uint32_t, 0, 0, true, 512, 512, 16, 8, 2, 0, true>(c, w0, w1, "pass1 early W8", r1);
    run<uint32_t, 0, 0, true, 512, 512, 16, 2, 2, 0, true>(c, w0, w1, "pass1 early W2", r1);
    std::swap(c.kA, c.kB);
    std::swap(c.vA, c.vB);
  }
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    std::vector<float> ts;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      CK(cudaMemcpyAsync(c.kB, c.kA, P * 8, cudaMemcpyDeviceToDevice));
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    printf("cudaMemcpy D2D of 16 B/pair: %.3f ms %.1f GB/s\n", ts[2], 16.0 * P / (ts[2] * 1e-3) / 1e9);
  }
  return 0;
}
