// Streaming bandwidth ceilings on this B200 (not product code): pure write,
// pure read and copy, 16-B and 32-B vector accesses, grid = k x 148 SMs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_write32(double* p, int64_t n4) {  // n4 = number of 32-B items
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    asm volatile("st.global.v4.f64 [%0], {%1, %1, %1, %1};" :: "l"(p + 4 * i), "d"(1.0) : "memory");
}
__global__ void k_write16(double2* p, int64_t n2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_double2(1.0, 2.0);
}
__global__ void k_read32(const double* p, int64_t n4, double* out) {
  double acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    double a, b, c, d;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p + 4 * i));
    acc += a + b + c + d;
  }
  if (acc == 12345.0) *out = acc;
}
__global__ void k_copy32(const double* s, double* d, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    double a, b, c, e;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(e) : "l"(s + 4 * i));
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" :: "l"(d + 4 * i), "d"(a), "d"(b), "d"(c), "d"(e) : "memory");
  }
}
int main() {
  const size_t bytes = (size_t)4 << 30;
  double *a, *b, *o;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&o, 64);
  cudaMemset(a, 0, bytes); cudaMemset(b, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int64_t n4 = bytes / 32;
  for (int mult : {2, 4, 8, 16}) {
    int grid = 148 * mult, th = 256;
    float ms;
    k_write32<<<grid, th>>>(a, n4);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k_write32<<<grid, th>>>(a, n4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("write32 grid %5d: %7.1f GB/s\n", grid, 5.0 * bytes / (ms * 1e-3) / 1e9);
    k_write16<<<grid, th>>>((double2*)a, bytes / 16);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k_write16<<<grid, th>>>((double2*)a, bytes / 16); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("write16 grid %5d: %7.1f GB/s\n", grid, 5.0 * bytes / (ms * 1e-3) / 1e9);
    k_read32<<<grid, th>>>(a, n4, o);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k_read32<<<grid, th>>>(a, n4, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("read32  grid %5d: %7.1f GB/s\n", grid, 5.0 * bytes / (ms * 1e-3) / 1e9);
    k_copy32<<<grid, th>>>(a, b, n4);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k_copy32<<<grid, th>>>(a, b, n4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("copy32  grid %5d: %7.1f GB/s (r+w)\n", grid, 10.0 * bytes / (ms * 1e-3) / 1e9);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
}
