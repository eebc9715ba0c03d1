// Synthetic-workload helper for the c4 dynamic-rebuild driver (not part of
// the build path): one fused pass x <- mod(x + N(0, scale^2), 1.0) over an
// f64 array, with np.mod's result convention (a tiny negative sum maps to
// exactly 1.0; zero stays +0.0).  Normals from Philox4x32-10 (counter =
// element quad index, key = seed ^ step) and Box-Muller in f32, so a
// trajectory is reproducible from (seed, step) alone.
#pragma once
#include "common.cuh"

namespace fmmb {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ double mod1(double v) {  // np.mod(v, 1.0) for v in (-1, 2)
  const double r = v - floor(v);  // exact for v in [0, 2); v + 1 rounded for v < 0
  return r == 0.0 ? 0.0 : r;      // -0.0 -> +0.0; a tiny negative v lands on 1.0
}

// Box-Muller pair from two 24-bit uniforms, in f32 (the noise is 1e-3 of a
// coordinate: f32's 2^-24 relative precision is 1e-10 absolute; tails are cut
// at 5.8 sigma)
__device__ __forceinline__ float2 normal_pair(uint32_t a, uint32_t b) {
  const float u1 = (float)((a >> 8) + 1u) * 0x1.0p-24f;  // (0, 1]
  const float u2 = (float)(b >> 8) * 0x1.0p-24f;         // [0, 1)
  const float rad = sqrtf(-2.0f * logf(u1));
  float s, c;
  sincospif(2.0f * u2, &s, &c);
  return make_float2(rad * c, rad * s);
}

// one Philox call (counter = quad index) perturbs four consecutive elements
__global__ void __launch_bounds__(256)
    k_perturb(double* __restrict__ x, int64_t n, uint64_t seed, uint64_t step, double scale) {
  const uint2 key = make_uint2((uint32_t)(seed ^ (step * 0x9E3779B97F4A7C15ull)),
                               (uint32_t)((seed >> 32) ^ step));
  const int64_t nquad = (n + 3) / 4;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nquad;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint4 r = philox4x32_10(make_uint4((uint32_t)p, (uint32_t)(p >> 32), 0u, 0u), key);
    const float2 g0 = normal_pair(r.x, r.y), g1 = normal_pair(r.z, r.w);
    const double d[4] = {(double)g0.x * scale, (double)g0.y * scale, (double)g1.x * scale,
                         (double)g1.y * scale};
    const int64_t i = 4 * p;
    if (i + 4 <= n && !(reinterpret_cast<uintptr_t>(x + i) & 31)) {
      double4 v = *reinterpret_cast<const double4*>(x + i);
      v.x = mod1(v.x + d[0]);
      v.y = mod1(v.y + d[1]);
      v.z = mod1(v.z + d[2]);
      v.w = mod1(v.w + d[3]);
      *reinterpret_cast<double4*>(x + i) = v;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i + k < n) x[i + k] = mod1(x[i + k] + d[k]);
    }
  }
}

}  // namespace fmmb

extern "C" fmmb_status fmmb_perturb(fmmb_handle_t h, double* x, int64_t n, uint64_t seed,
                                    uint64_t step, double scale, void* stream) {
  FMMB_GUARD(h);
  if (n < 0 || (n > 0 && !x)) return FMMB_ERR_ARG;
  cudaSetDevice(h->device);
  if (n == 0) return FMMB_OK;
  const int64_t quads = (n + 3) / 4;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((quads + 255) / 256,
                                                               (int64_t)h->num_sms * 16));
  fmmb::k_perturb<<<grid, 256, 0, (cudaStream_t)stream>>>(x, n, seed, step, scale);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fmmb_fail(h, FMMB_ERR_CUDA, "perturb: %s", cudaGetErrorString(e));
  return FMMB_OK;
}
