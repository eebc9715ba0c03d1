// Micro-benchmarks for the scatter design (not product code):
//  A: random atomicAdd(+1) on NB padded cursors, K independent per thread in flight
//  B: same, then a dependent 32-B store to the returned slot
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
template <int K, bool STORE>
__global__ void k_atom(uint32_t* cursor, int stride, int nbm1, double* rec, int64_t total) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = t; i < total; i += nthreads * K) {
    uint32_t slot[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      uint32_t b = hash32((uint32_t)(i + k * nthreads)) & nbm1;
      slot[k] = atomicAdd(cursor + (size_t)b * stride, 1u);
    }
    if (STORE) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double* p = rec + 4 * (size_t)(slot[k] & ((1u << 25) - 1));
        asm volatile("st.global.v4.f64 [%0], {%1, %1, %1, %1};" :: "l"(p), "d"(1.0) : "memory");
      }
    } else {
      uint32_t acc = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) acc += slot[k];
      if (acc == 0xFFFFFFFFu) cursor[0] = acc;
    }
  }
}
int main() {
  const int64_t total = 1 << 25;
  uint32_t* cursor; double* rec;
  cudaMalloc(&cursor, (size_t)32768 * 32 * 4);
  cudaMalloc(&rec, (size_t)total * 32);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto kern, int stride, int nb, int blocks, int threads) {
    cudaMemset(cursor, 0, (size_t)32768 * 32 * 4);
    kern<<<blocks, threads>>>(cursor, stride, nb - 1, rec, total);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) kern<<<blocks, threads>>>(cursor, stride, nb - 1, rec, total);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-28s stride %2d nb %6d grid %5d x %4d: %8.1f us  (%.2f Gatom/s)\n", name, stride, nb, blocks,
           threads, ms / 3 * 1e3, total / (ms / 3 * 1e-3) / 1e9);
  };
  for (int stride : {1, 8, 32})
    for (int nb : {4096, 32768}) {
      run("atom K=1", k_atom<1, false>, stride, nb, 148 * 4, 512);
      run("atom K=4", k_atom<4, false>, stride, nb, 148 * 4, 512);
      run("atom K=8", k_atom<8, false>, stride, nb, 148 * 4, 512);
    }
  run("atom+store K=1", k_atom<1, true>, 32, 32768, 148 * 4, 512);
  run("atom+store K=4", k_atom<4, true>, 32, 32768, 148 * 4, 512);
  run("atom+store K=8", k_atom<8, true>, 32, 32768, 148 * 4, 512);
  run("atom+store K=8 2k", k_atom<8, true>, 32, 32768, 148 * 2, 1024);
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
