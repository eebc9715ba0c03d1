// Store-pattern micro-benchmark for the list writer (not product code):
// every warp streams a private contiguous region (like CSR rows), with
// k of 32 lanes active per instruction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int ACTIVE, bool CODES, bool RANKS>
__global__ void k_stream(int64_t* r, int16_t* c, int64_t per_warp) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t* rp = r + w * per_warp;
  int16_t* cp = c + w * per_warp;
  for (int64_t o = 0; o + ACTIVE <= per_warp; o += ACTIVE) {
    if (lane < ACTIVE) {
      if (RANKS) rp[o + lane] = o + lane;
      if (CODES) cp[o + lane] = (int16_t)lane;
    }
  }
}
// 16-B vector stores of a warp-contiguous stream
__global__ void k_stream16(int64_t* r, int64_t per_warp) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  longlong2* rp = reinterpret_cast<longlong2*>(r + w * per_warp);
  for (int64_t o = 0; o + 32 <= per_warp / 2; o += 32) rp[o + lane] = make_longlong2(o, lane);
}
// rows produced 26 entries at a time (ballot-compacted), staged in shared
// memory and flushed as 16-B vectors: ranks 64 per flush, codes 256 per flush
__global__ void k_staged(int64_t* r, int16_t* c, int64_t per_warp) {
  __shared__ __align__(16) int64_t sr[8][128];
  __shared__ __align__(16) int16_t sc[8][512];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t* rp = r + w * per_warp;
  int16_t* cp = c + w * per_warp;
  int nr = 0, nc = 0;       // staged counts
  int64_t fr = 0, fc = 0;   // flushed
  for (int64_t o = 0; o + 26 <= per_warp; o += 26) {
    if (lane < 26) {
      sr[warp][(nr + lane) & 127] = o + lane;
      sc[warp][(nc + lane) & 511] = (int16_t)lane;
    }
    nr += 26; nc += 26;
    __syncwarp();
    if (nr - fr >= 64) {  // 64 ranks = 32 lanes x 16 B
      const int at = (int)(fr & 127);
      reinterpret_cast<longlong2*>(rp + fr)[lane] = reinterpret_cast<const longlong2*>(&sr[warp][at])[lane];
      fr += 64;
    }
    if (nc - fc >= 256) {  // 256 codes = 32 lanes x 16 B
      const int at = (int)(fc & 511);
      reinterpret_cast<int4*>(cp + fc)[lane] = reinterpret_cast<const int4*>(&sc[warp][at])[lane];
      fc += 256;
    }
    __syncwarp();
  }
}

// rows of 184 entries produced 23 lanes x 8 chunks into shared memory
// (st.shared, ranks + codes), flushed by one TMA bulk store per stream per
// row (cp.async.bulk.global.shared::cta), double-buffered per warp
__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
template <int WARPS>
__global__ void k_tma(int64_t* r, int16_t* c, int64_t per_warp) {
  __shared__ __align__(128) int64_t sr[WARPS][2][184];
  __shared__ __align__(128) int16_t sc[WARPS][2][184];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t* rp = r + w * per_warp;
  int16_t* cp = c + w * per_warp;
  int buf = 0;
  for (int64_t o = 0; o + 184 <= per_warp; o += 184, buf ^= 1) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int ch = 0; ch < 8; ++ch)
      if (lane < 23) {
        sr[warp][buf][ch * 23 + lane] = o + ch * 23 + lane;
        sc[warp][buf][ch * 23 + lane] = (int16_t)lane;
      }
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(rp + o),
                   "r"(s_u32(&sr[warp][buf][0])), "r"(184 * 8) : "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(cp + o),
                   "r"(s_u32(&sc[warp][buf][0])), "r"(184 * 2) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
int main() {
  const int64_t N = (int64_t)1 << 29;  // 4 GiB of i64
  int64_t* r; int16_t* c;
  cudaMalloc(&r, N * 8); cudaMalloc(&c, N * 2);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, int grid, int block, double bytes, auto... args) {
    kern<<<grid, block>>>(args...);
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) kern<<<grid, block>>>(args...);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s grid %5d: %8.1f us  %7.1f GB/s\n", name, grid, ms / 3 * 1e3, bytes / (ms / 3 * 1e-3) / 1e9);
  };
  for (int grid : {148 * 8, 148 * 16, 148 * 32}) {
    const int64_t warps = (int64_t)grid * 8;
    const int64_t per = (N / warps) & ~(int64_t)255;
    run("rank i64, 32 lanes", k_stream<32, false, true>, grid, 256, 8.0 * N, r, c, per);
    run("rank i64, 26 lanes", k_stream<26, false, true>, grid, 256, 8.0 * (per / 26 * 26) * warps, r, c, per);
    run("code i16, 26 lanes", k_stream<26, true, false>, grid, 256, 2.0 * (per / 26 * 26) * warps, r, c, per);
    run("rank+code, 26 lanes", k_stream<26, true, true>, grid, 256, 10.0 * (per / 26 * 26) * warps, r, c, per);
    run("rank 16B vectors", k_stream16, grid, 256, 8.0 * (per / 64 * 64) * warps, r, per);
    run("rank+code staged, 16B flushes", k_staged, grid, 256, 10.0 * (per / 26 * 26) * warps, r, c, per);
    run("rank+code TMA bulk rows (184)", k_tma<8>, grid, 256, 10.0 * (per / 184 * 184) * warps, r, c, per);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
