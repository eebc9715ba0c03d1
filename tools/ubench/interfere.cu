// Micro-benchmark (not product code): is the build L2-request bound?  The
// bucket scatter (random 32-B record stores + cursor atomics) runs alone and
// concurrently with a 4.8 GB streaming write issued as (0) per-lane 8-B + 2-B
// stores (the list writer's pattern), (1) 32-B per lane vector stores (1 KB
// per warp instruction), (2) TMA bulk stores of 4 KB from shared memory.
// If the pair's time is the sum of the parts for (0) but closer to the max
// for (1)/(2), the shared bottleneck is L2 requests, not DRAM bytes.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

constexpr int L = 7, SB = 3 * L, BB = 14, SHIFT = SB - BB, NB = 2 << BB;
__device__ __forceinline__ uint64_t dil(uint64_t v) {
  v &= 0x1FFFFFull;
  v = (v | (v << 32)) & 0x001F00000000FFFFull;
  v = (v | (v << 16)) & 0x001F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__global__ void __launch_bounds__(512) k_scat(const double* pts, int64_t n, int64_t tot,
                                              uint32_t* cursor, double* rec,
                                              unsigned long long* bmp) {
  constexpr int IT = 4;
  const int64_t stride = (int64_t)gridDim.x * 512 * IT;
  for (int64_t base = (int64_t)blockIdx.x * 512 * IT; base < tot; base += stride) {
    double x[IT], y[IT], z[IT];
    uint32_t slot[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int64_t i = base + k * 512 + threadIdx.x;
      if (i < tot) { x[k] = pts[3 * i]; y[k] = pts[3 * i + 1]; z[k] = pts[3 * i + 2]; }
    }
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int64_t i = base + k * 512 + threadIdx.x;
      if (i < tot) {
        const double g = 128.0;
        const uint32_t key = (uint32_t)(dil((uint64_t)(x[k] * g)) | (dil((uint64_t)(y[k] * g)) << 1) |
                                        (dil((uint64_t)(z[k] * g)) << 2));
        asm volatile("red.global.or.b64 [%0], %1;" ::"l"(bmp + (i >= n ? (1 << SB) / 64 : 0) + (key >> 6)),
                     "l"(1ull << (key & 63)) : "memory");
        slot[k] = atomicAdd(cursor + (size_t)(((i >= n) << BB) | (key >> SHIFT)) * 32, 1u);
      }
    }
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int64_t i = base + k * 512 + threadIdx.x;
      if (i < tot)
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(rec + 4 * (size_t)slot[k]),
                     "d"(x[k]), "d"(y[k]), "d"(z[k]), "d"(x[k]) : "memory");
    }
  }
}

// streaming writer: every warp owns a contiguous region of ranks (i64) and codes (i16)
template <int MODE>
__global__ void __launch_bounds__(256) k_wr(int64_t* r, int16_t* c, int64_t per_warp) {
  __shared__ __align__(128) int64_t sr[8][2][256];
  __shared__ __align__(128) int16_t sc[8][2][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t* rp = r + w * per_warp;
  int16_t* cp = c + w * per_warp;
  if (MODE == 0) {
    for (int64_t o = 0; o + 32 <= per_warp; o += 32) {
      rp[o + lane] = o + lane;
      cp[o + lane] = (int16_t)lane;
    }
  } else if (MODE == 1) {
    for (int64_t o = 0; o + 128 <= per_warp; o += 128) {
      asm volatile("st.global.v4.b64 [%0], {%1, %1, %1, %1};" ::"l"(rp + o + 4 * lane), "l"(o) : "memory");
      if ((o & 511) == 0 && o + 512 <= per_warp)
        asm volatile("st.global.v4.b64 [%0], {%1, %1, %1, %1};" ::"l"(cp + o + 16 * lane), "l"(o) : "memory");
    }
  } else {
    int buf = 0;
    for (int64_t o = 0; o + 256 <= per_warp; o += 256, buf ^= 1) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      for (int k = lane; k < 256; k += 32) { sr[warp][buf][k] = o + k; sc[warp][buf][k] = (int16_t)k; }
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(rp + o),
                     "r"((uint32_t)__cvta_generic_to_shared(&sr[warp][buf][0])), "r"(256 * 8) : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(cp + o),
                     "r"((uint32_t)__cvta_generic_to_shared(&sc[warp][buf][0])), "r"(256 * 2) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const int64_t n = 1 << 24, tot = 2 * n;
  std::vector<double> h(3 * tot);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  for (auto& v : h) v = U(rng);
  double *pts, *rec;
  uint32_t* cursor;
  unsigned long long* bmp;
  cudaMalloc(&pts, 8 * 3 * tot);
  cudaMalloc(&rec, (size_t)32 * NB * 2600);
  cudaMalloc(&cursor, (size_t)NB * 32 * 4);
  cudaMalloc(&bmp, 2 * (1 << SB) / 8);
  cudaMemcpy(pts, h.data(), 8 * 3 * tot, cudaMemcpyHostToDevice);
  std::vector<uint32_t> hc((size_t)NB * 32, 0);
  for (int b = 0; b < NB; ++b) hc[(size_t)b * 32] = (uint32_t)b * 2600;
  const int64_t N = 480000000;  // 4.8 GB of ranks + codes (10 B per entry)
  int64_t* r;
  int16_t* c;
  cudaMalloc(&r, N * 8 + 4096);
  cudaMalloc(&c, N * 2 + 4096);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  const int wgrid = 148 * 4;
  const int64_t per = (N / ((int64_t)wgrid * 8)) & ~(int64_t)511;
  uint32_t* cursor0;
  cudaMalloc(&cursor0, hc.size() * 4);
  cudaMemcpy(cursor0, hc.data(), hc.size() * 4, cudaMemcpyHostToDevice);
  auto scat = [&](cudaStream_t s) {
    cudaMemcpyAsync(cursor, cursor0, hc.size() * 4, cudaMemcpyDeviceToDevice, s);
    k_scat<<<148 * 2, 512, 0, s>>>(pts, n, tot, cursor, rec, bmp);
  };
  auto wr = [&](int mode, cudaStream_t s) {
    if (mode == 0) k_wr<0><<<wgrid, 256, 0, s>>>(r, c, per);
    if (mode == 1) k_wr<1><<<wgrid, 256, 0, s>>>(r, c, per);
    if (mode == 2) k_wr<2><<<wgrid, 256, 0, s>>>(r, c, per);
  };
  auto timed = [&](auto f) {
    f();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0, s1);
      cudaStreamWaitEvent(s2, e0, 0);
      f();
      cudaEventRecord(e2, s2);
      cudaStreamWaitEvent(s1, e2, 0);
      cudaEventRecord(e1, s1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    return best * 1e3f;
  };
  const float ts = timed([&] { scat(s1); });
  printf("scatter alone: %8.1f us\n", ts);
  const char* names[3] = {"per-lane 8B+2B", "v4 32B/lane", "TMA bulk 2KB"};
  for (int mode = 0; mode < 3; ++mode) {
    const float tw = timed([&] { wr(mode, s2); });
    const float tb = timed([&] { scat(s1); wr(mode, s2); });
    printf("write %-16s alone %8.1f us (%6.0f GB/s) | with scatter %8.1f us (sum %8.1f, max %8.1f)\n",
           names[mode], tw, 10.0 * per * wgrid * 8 / (tw * 1e-6) / 1e9, tb, tw + ts, tw > ts ? tw : ts);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
