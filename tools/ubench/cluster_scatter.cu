// Micro-benchmark (not product code): bucket scatter with slot claims on
// global L2 cursors vs cluster-private bucket regions whose cursors live in
// distributed shared memory (DSMEM atomics, no L2 operation per claim), and
// the occupancy bitmap built in DSMEM vs red.global.or.  c2 geometry:
// 2^25 points, L = 7, 2 x 2^14 buckets (top 14 of 21 key bits + set bit).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int L = 7, SB = 3 * L, BB = 14, SHIFT = SB - BB, NB = 2 << BB;
constexpr int TPB = 512, ITEMS = 4;
__device__ __forceinline__ uint64_t dil(uint64_t v) {
  v &= 0x1FFFFFull;
  v = (v | (v << 32)) & 0x001F00000000FFFFull;
  v = (v | (v << 16)) & 0x001F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__device__ __forceinline__ uint32_t key_of(const double* p) {
  const double g = (double)(1 << L);
  uint64_t ix = (uint64_t)(long long)(p[0] * g), iy = (uint64_t)(long long)(p[1] * g),
           iz = (uint64_t)(long long)(p[2] * g);
  return (uint32_t)(dil(ix) | (dil(iy) << 1) | (dil(iz) << 2));
}
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}

// ---- global cursors (the current design, without the TMA ring)
template <bool OCC>
__global__ void __launch_bounds__(TPB) k_glob(const double* pts, int64_t n, int64_t tot,
                                              uint32_t* cursor, double* rec,
                                              unsigned long long* bmp) {
  const int64_t stride = (int64_t)gridDim.x * TPB * ITEMS;
  for (int64_t base = (int64_t)blockIdx.x * TPB * ITEMS; base < tot; base += stride) {
    double x[ITEMS], y[ITEMS], z[ITEMS];
    uint32_t slot[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < tot) {
        x[k] = pts[3 * i]; y[k] = pts[3 * i + 1]; z[k] = pts[3 * i + 2];
      }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < tot) {
        double p[3] = {x[k], y[k], z[k]};
        const uint32_t key = key_of(p);
        if (OCC)
          asm volatile("red.global.or.b64 [%0], %1;" ::"l"(bmp + (i >= n ? (1 << SB) / 64 : 0) + (key >> 6)),
                       "l"(1ull << (key & 63)) : "memory");
        const uint32_t b = ((i >= n) << BB) | (key >> SHIFT);
        slot[k] = atomicAdd(cursor + (size_t)b * 32, 1u);
      }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < tot) st4(rec + 4 * (size_t)slot[k], x[k], y[k], z[k], __longlong_as_double(i));
    }
  }
}

// ---- cluster-private regions, cursors in DSMEM (bucket b lives in CTA b % CS)
template <int CS>
__global__ void __launch_bounds__(TPB) k_clus(const double* pts, int64_t n, int64_t tot,
                                              int64_t chunk, const uint32_t* off, int G,
                                              double* rec) {
  extern __shared__ uint32_t s_cur[];  // [NB / CS]
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int c = blockIdx.x / CS;
  for (int j = threadIdx.x; j < NB / CS; j += TPB) s_cur[j] = off[(size_t)(j * CS + r) * G + c];
  cl.sync();
  const int64_t lo = (int64_t)c * chunk, hi = lo + chunk < tot ? lo + chunk : tot;
  for (int64_t base = lo + (int64_t)r * TPB * ITEMS; base < hi; base += (int64_t)CS * TPB * ITEMS) {
    double x[ITEMS], y[ITEMS], z[ITEMS];
    uint32_t slot[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < hi) {
        x[k] = pts[3 * i]; y[k] = pts[3 * i + 1]; z[k] = pts[3 * i + 2];
      }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < hi) {
        double p[3] = {x[k], y[k], z[k]};
        const uint32_t key = key_of(p);
        const uint32_t b = ((i >= n) << BB) | (key >> SHIFT);
        uint32_t* rc = cl.map_shared_rank(s_cur + b / CS, (int)(b % CS));
        slot[k] = atomicAdd(rc, 1u);
      }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < hi) st4(rec + 4 * (size_t)slot[k], x[k], y[k], z[k], __longlong_as_double(i));
    }
  }
  cl.sync();
}

// ---- cluster histogram (+ occupancy bitmap) in DSMEM
template <int CS, bool OCC>
__global__ void __launch_bounds__(TPB) k_chist(const double* pts, int64_t n, int64_t tot,
                                               int64_t chunk, uint32_t* hist, int G,
                                               unsigned long long* bmp) {
  extern __shared__ uint32_t s_h[];  // [NB / CS] counts | [2 * 2^SB / 32 / CS] bitmap words
  constexpr int HW = NB / CS;
  constexpr int BW = 2 * (1 << SB) / 32 / CS;
  uint32_t* s_b = s_h + HW;
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int c = blockIdx.x / CS;
  for (int j = threadIdx.x; j < HW; j += TPB) s_h[j] = 0;
  if (OCC)
    for (int j = threadIdx.x; j < BW; j += TPB) s_b[j] = 0;
  cl.sync();
  const int64_t lo = (int64_t)c * chunk, hi = lo + chunk < tot ? lo + chunk : tot;
  for (int64_t base = lo + (int64_t)r * TPB * ITEMS; base < hi; base += (int64_t)CS * TPB * ITEMS) {
    double x[ITEMS], y[ITEMS], z[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < hi) {
        x[k] = pts[3 * i]; y[k] = pts[3 * i + 1]; z[k] = pts[3 * i + 2];
      }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < hi) {
        double p[3] = {x[k], y[k], z[k]};
        const uint32_t key = key_of(p);
        const uint32_t b = ((i >= n) << BB) | (key >> SHIFT);
        atomicAdd(cl.map_shared_rank(s_h + b / CS, (int)(b % CS)), 1u);
        if (OCC) {
          // bitmap word w (32-bit) of the combined [src | recv] bitmap, word-interleaved over CTAs
          const uint32_t w = ((uint32_t)(i >= n) << (SB - 5)) | (key >> 5);
          atomicOr(cl.map_shared_rank(s_b + w / CS, (int)(w % CS)), 1u << (key & 31));
        }
      }
    }
  }
  cl.sync();
  for (int j = threadIdx.x; j < HW; j += TPB) hist[(size_t)c * NB + j * CS + r] = s_h[j];
  if (OCC)
    for (int j = threadIdx.x; j < BW; j += TPB) {
      const uint32_t v = s_b[j];
      if (v) atomicOr(reinterpret_cast<unsigned*>(bmp) + j * CS + r, v);
    }
}

// ---- per-CTA smem histogram (the current k_bkt_hist shape), + red.global.or occupancy
template <bool OCC>
__global__ void __launch_bounds__(TPB) k_ghist(const double* pts, int64_t n, int64_t tot,
                                               uint32_t* hist, unsigned long long* bmp) {
  extern __shared__ uint32_t s_h[];
  for (int j = threadIdx.x; j < NB; j += TPB) s_h[j] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * TPB * ITEMS;
  for (int64_t base = (int64_t)blockIdx.x * TPB * ITEMS; base < tot; base += stride) {
    double x[ITEMS], y[ITEMS], z[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < tot) {
        x[k] = pts[3 * i]; y[k] = pts[3 * i + 1]; z[k] = pts[3 * i + 2];
      }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < tot) {
        double p[3] = {x[k], y[k], z[k]};
        const uint32_t key = key_of(p);
        atomicAdd(s_h + (((i >= n) << BB) | (key >> SHIFT)), 1u);
        if (OCC)
          asm volatile("red.global.or.b64 [%0], %1;" ::"l"(bmp + (i >= n ? (1 << SB) / 64 : 0) + (key >> 6)),
                       "l"(1ull << (key & 63)) : "memory");
      }
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < NB; j += TPB) hist[(size_t)blockIdx.x * NB + j] = s_h[j];
}


// ---- CTA-private bucket regions (exact offsets from the per-CTA histogram),
// cursors in the CTA's own shared memory (no L2 operation per claim)
template <bool OCC>
__global__ void __launch_bounds__(TPB) k_ctas(const double* pts, int64_t n, int64_t tot,
                                              const uint32_t* off, int G, double* rec,
                                              unsigned long long* bmp) {
  extern __shared__ uint32_t s_cur[];  // [NB]
  for (int j = threadIdx.x; j < NB; j += TPB) s_cur[j] = off[(size_t)j * G + blockIdx.x];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * TPB * ITEMS;
  for (int64_t base = (int64_t)blockIdx.x * TPB * ITEMS; base < tot; base += stride) {
    double x[ITEMS], y[ITEMS], z[ITEMS];
    uint32_t slot[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < tot) {
        x[k] = pts[3 * i]; y[k] = pts[3 * i + 1]; z[k] = pts[3 * i + 2];
      }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < tot) {
        double p[3] = {x[k], y[k], z[k]};
        const uint32_t key = key_of(p);
        if (OCC)
          asm volatile("red.global.or.b64 [%0], %1;" ::"l"(bmp + (i >= n ? (1 << SB) / 64 : 0) + (key >> 6)),
                       "l"(1ull << (key & 63)) : "memory");
        slot[k] = atomicAdd(s_cur + (((i >= n) << BB) | (key >> SHIFT)), 1u);
      }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t i = base + k * TPB + threadIdx.x;
      if (i < tot) st4(rec + 4 * (size_t)slot[k], x[k], y[k], z[k], __longlong_as_double(i));
    }
  }
}

template <typename K, typename... A>
float time_launch(K kern, int grid, int cs, size_t smem, int reps, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TPB);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, kern, args...);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, kern, args...);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("  error: %s\n", cudaGetErrorString(e));
  return ms / reps * 1e3f;
}

template <int CS>
void run_cluster(const double* pts, int64_t n, int64_t tot, double* rec, uint32_t* dhist,
                 uint32_t* doff, unsigned long long* bmp) {
  auto kh = k_chist<CS, true>;
  auto kh0 = k_chist<CS, false>;
  auto ks = k_clus<CS>;
  const size_t hsm = (NB / CS + 2 * (1 << SB) / 32 / CS) * 4, ssm = NB / CS * 4;
  for (auto k : {kh, kh0}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
    if (CS > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
  if (CS > 8) cudaFuncSetAttribute(ks, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  // clusters resident at once
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS * 64);
  cfg.blockDim = dim3(TPB);
  cfg.dynamicSmemBytes = ssm;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim = {(unsigned)CS, 1, 1};
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  cudaOccupancyMaxActiveClusters(&ncl, ks, &cfg);
  cfg.dynamicSmemBytes = hsm;
  int nclh = 0;
  cudaOccupancyMaxActiveClusters(&nclh, kh, &cfg);
  const int G = ncl;  // scatter and histogram share the cluster -> chunk map
  const int64_t chunk = (tot + G - 1) / G;
  float th = time_launch(kh, G * CS, CS, hsm, 5, pts, n, tot, chunk, dhist, G, bmp);
  float th0 = time_launch(kh0, G * CS, CS, hsm, 5, pts, n, tot, chunk, dhist, G, bmp);
  // region offsets, bucket-major then cluster
  std::vector<uint32_t> h((size_t)G * NB), off((size_t)NB * G);
  cudaMemcpy(h.data(), dhist, h.size() * 4, cudaMemcpyDeviceToHost);
  uint64_t run = 0;
  for (int b = 0; b < NB; ++b)
    for (int c = 0; c < G; ++c) {
      off[(size_t)b * G + c] = (uint32_t)run;
      run += h[(size_t)c * NB + b];
    }
  cudaMemcpy(doff, off.data(), off.size() * 4, cudaMemcpyHostToDevice);
  float ts = time_launch(ks, G * CS, CS, ssm, 5, pts, n, tot, chunk, (const uint32_t*)doff, G, rec);
  printf("CS %2d: clusters %3d (hist-shape %3d), total %llu | chist+occ %7.1f us, chist %7.1f us, "
         "cluster scatter %7.1f us\n",
         CS, G, nclh, (unsigned long long)run, th, th0, ts);
}

int main() {
  const int64_t n = 1 << 24, m = 1 << 24, tot = n + m;
  std::vector<double> h(3 * tot);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  for (auto& v : h) v = U(rng);
  double *pts, *rec;
  uint32_t *cursor, *hist, *off;
  unsigned long long* bmp;
  cudaMalloc(&pts, 8 * 3 * tot);
  cudaMalloc(&rec, (size_t)32 * NB * 2600 + 4096);
  cudaMalloc(&cursor, (size_t)NB * 32 * 4);
  cudaMalloc(&hist, (size_t)NB * 4 * 1024);
  cudaMalloc(&off, (size_t)NB * 4 * 1024);
  cudaMalloc(&bmp, 2 * (1 << SB) / 8);
  cudaMemcpy(pts, h.data(), 8 * 3 * tot, cudaMemcpyHostToDevice);
  // global-cursor scatter: cursors seeded with exact-enough regions
  std::vector<uint32_t> hc((size_t)NB * 32, 0);
  for (int b = 0; b < NB; ++b) hc[(size_t)b * 32] = (uint32_t)b * 2600;
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per_sm : {2, 4}) {
    cudaMemcpy(cursor, hc.data(), hc.size() * 4, cudaMemcpyHostToDevice);
    float t0 = time_launch(k_glob<false>, dev_sms * per_sm, 1, 0, 1, pts, n, tot, cursor, rec, bmp);
    cudaMemcpy(cursor, hc.data(), hc.size() * 4, cudaMemcpyHostToDevice);
    float t1 = time_launch(k_glob<true>, dev_sms * per_sm, 1, 0, 1, pts, n, tot, cursor, rec, bmp);
    printf("global cursors, %d CTA/SM: scatter %7.1f us, scatter+occ %7.1f us\n", per_sm, t0, t1);
  }
  cudaFuncSetAttribute(k_ghist<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * 4);
  cudaFuncSetAttribute(k_ghist<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * 4);
  printf("per-CTA smem hist: %7.1f us, + red.global.or occ %7.1f us\n",
         time_launch(k_ghist<false>, dev_sms, 1, NB * 4, 5, pts, n, tot, hist, bmp),
         time_launch(k_ghist<true>, dev_sms, 1, NB * 4, 5, pts, n, tot, hist, bmp));
  {  // CTA-private regions: per-CTA histogram -> bucket-major offsets -> smem cursors
    const int G = dev_sms;
    time_launch(k_ghist<false>, G, 1, NB * 4, 1, pts, n, tot, hist, bmp);
    std::vector<uint32_t> hh((size_t)G * NB), oo((size_t)NB * G);
    cudaMemcpy(hh.data(), hist, hh.size() * 4, cudaMemcpyDeviceToHost);
    uint64_t run = 0;
    for (int b = 0; b < NB; ++b)
      for (int c = 0; c < G; ++c) {
        oo[(size_t)b * G + c] = (uint32_t)run;
        run += hh[(size_t)c * NB + b];
      }
    cudaMemcpy(off, oo.data(), oo.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_ctas<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * 4);
    cudaFuncSetAttribute(k_ctas<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * 4);
    printf("CTA-private regions (%d CTAs, total %llu): scatter %7.1f us, scatter+occ %7.1f us\n", G,
           (unsigned long long)run,
           time_launch(k_ctas<false>, G, 1, NB * 4, 5, pts, n, tot, (const uint32_t*)off, G, rec, bmp),
           time_launch(k_ctas<true>, G, 1, NB * 4, 5, pts, n, tot, (const uint32_t*)off, G, rec, bmp));
  }
  run_cluster<4>(pts, n, tot, rec, hist, off, bmp);
  run_cluster<8>(pts, n, tot, rec, hist, off, bmp);
  run_cluster<16>(pts, n, tot, rec, hist, off, bmp);
  return 0;
}
