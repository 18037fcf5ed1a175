// bench_atomics.cu — developer tool: throughput of global atomics indexed by mesh node ids
// (counting-sort transpose feasibility).  Kuhn n^3 tets in natural order and randomly relabelled.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__global__ void gen_kuhn(int n, int32_t* conn) {
  const int64_t ncell = (int64_t)n * n * n;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ci = c % n, cj = (c / n) % n, ck = c / ((int64_t)n * n), w = n + 1;
    const int64_t base = ci + w * (cj + w * ck), step[3] = {1, w, w * w};
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int p = 0; p < 6; ++p) {
      int32_t* t = conn + (c * 6 + p) * 4;
      t[0] = (int32_t)base; t[1] = (int32_t)(base + step[perms[p][0]]);
      t[2] = (int32_t)(base + step[perms[p][0]] + step[perms[p][1]]); t[3] = (int32_t)(base + 1 + w + w * w);
    }
  }
}
__global__ void scramble(int32_t* conn, int64_t n, int64_t N) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    conn[i] = (int32_t)(((uint64_t)conn[i] * 2654435761ull) % (uint64_t)N);
}
// count: one RED per incidence (int4 loads of a tet row)
__global__ void k_count(const int4* conn, int64_t M, int* cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M; e += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = conn[e];
    atomicAdd(cnt + r.x, 1); atomicAdd(cnt + r.y, 1); atomicAdd(cnt + r.z, 1); atomicAdd(cnt + r.w, 1);
  }
}
// scatter: returning atomic cursor per incidence, write element id to off[node] + slot
__global__ void k_scatter(const int4* conn, int64_t M, const long long* off, int* cur, int* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M; e += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = conn[e];
    const int a = atomicAdd(cur + r.x, 1), b = atomicAdd(cur + r.y, 1), c = atomicAdd(cur + r.z, 1), d = atomicAdd(cur + r.w, 1);
    out[off[r.x] + a] = (int)e; out[off[r.y] + b] = (int)e; out[off[r.z] + c] = (int)e; out[off[r.w] + d] = (int)e;
  }
}
__global__ void k_prefix_naive(const int* cnt, int64_t N, long long* off) {   // placeholder offsets: i*24 spacing
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) off[i] = i * 32;
}
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 320;
  const int64_t M = 6LL * n * n * n, N = (int64_t)(n + 1) * (n + 1) * (n + 1);
  int32_t* conn; int* cnt; long long* off; int* out;
  CK(cudaMalloc(&conn, M * 16)); CK(cudaMalloc(&cnt, N * 4)); CK(cudaMalloc(&off, N * 8)); CK(cudaMalloc(&out, N * 32 * 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int scr = 0; scr < 2; ++scr) {
    gen_kuhn<<<148 * 8, 256>>>(n, conn);
    if (scr) scramble<<<148 * 8, 256>>>(conn, M * 4, N);
    k_prefix_naive<<<148 * 8, 256>>>(cnt, N, off);
    CK(cudaDeviceSynchronize());
    for (int grid : {148 * 8, 148 * 32}) {
      std::vector<float> tc, ts;
      for (int r = 0; r < 5; ++r) {
        CK(cudaMemset(cnt, 0, N * 4));
        cudaEventRecord(e0); k_count<<<grid, 256>>>((const int4*)conn, M, cnt); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); tc.push_back(ms);
        CK(cudaMemset(cnt, 0, N * 4));
        cudaEventRecord(e0); k_scatter<<<grid, 256>>>((const int4*)conn, M, off, cnt, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms);
      }
      std::sort(tc.begin(), tc.end()); std::sort(ts.begin(), ts.end());
      printf("%s grid=%d: count %.3f ms (%.1f G atomics/s)  scatter %.3f ms (%.1f G/s)\n", scr ? "random " : "natural", grid,
             tc[2], 4.0 * M / tc[2] / 1e6, ts[2], 4.0 * M / ts[2] / 1e6);
    }
  }
  return 0;
}
