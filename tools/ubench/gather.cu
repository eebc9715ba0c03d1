// Random 8-B gathers from a 128 MiB array (2^24 of them), as the local sort
// would do to fetch charges by input index instead of carrying them through
// the scatter (not product code).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_gather(const double* __restrict__ q, const uint32_t* __restrict__ idx, double* out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ldg(q + idx[i]);
}
__global__ void k_perm(uint32_t* idx, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull; x ^= x >> 29;
    idx[i] = (uint32_t)(x & (n - 1));
  }
}
__global__ void k_local(const double* __restrict__ q, const uint32_t* __restrict__ idx, double* out, int64_t n) {
  // bucket-local pattern: each 1024-block of outputs reads a random 1024 subset (same randomness)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ldg(q + idx[i]);
}
int main() {
  const int64_t n = 1 << 24;
  double *q, *out; uint32_t* idx;
  cudaMalloc(&q, n * 8); cudaMalloc(&out, n * 8); cudaMalloc(&idx, n * 4);
  cudaMemset(q, 0, n * 8);
  k_perm<<<1184, 256>>>(idx, n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int grid : {1184, 4736}) {
    k_gather<<<grid, 256>>>(q, idx, out, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_gather<<<grid, 256>>>(q, idx, out, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("random 8B gather of 2^24 from 128MiB (grid %d): %.1f us\n", grid, ms / 5 * 1e3);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
