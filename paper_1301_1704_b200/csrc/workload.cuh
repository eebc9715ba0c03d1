// Synthetic-workload helper for the c4 dynamic-rebuild driver (not part of
// the build path): one fused pass x <- mod(x + N(0, scale^2), 1.0) over an
// f64 array, with np.mod's result convention (a tiny negative sum maps to
// exactly 1.0; zero stays +0.0).  Normals from Philox4x32-10 (counter =
// element pair index, key = seed ^ step) and Box-Muller in f64, so a
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

__device__ __forceinline__ double mod1(double v) {  // np.mod(v, 1.0)
  double r = fmod(v, 1.0);
  if (r != 0.0 && r < 0.0) r += 1.0;
  return r == 0.0 ? 0.0 : r;
}

__global__ void __launch_bounds__(256)
    k_perturb(double* __restrict__ x, int64_t n, uint64_t seed, uint64_t step, double scale) {
  const uint2 key = make_uint2((uint32_t)(seed ^ (step * 0x9E3779B97F4A7C15ull)),
                               (uint32_t)((seed >> 32) ^ step));
  const int64_t npair = (n + 1) / 2;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npair;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint4 r = philox4x32_10(make_uint4((uint32_t)p, (uint32_t)(p >> 32), 0u, 0u), key);
    // two uniforms in (0, 1] with 53 random bits each
    const double u1 = ((double)((((uint64_t)r.x << 32) | r.y) >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)((((uint64_t)r.z << 32) | r.w) >> 11) * 0x1.0p-53;
    const double rad = sqrt(-2.0 * log(u1)) * scale;
    double s, c;
    sincospi(2.0 * u2, &s, &c);
    const int64_t i = 2 * p;
    x[i] = mod1(x[i] + rad * c);
    if (i + 1 < n) x[i + 1] = mod1(x[i + 1] + rad * s);
  }
}

}  // namespace fmmb

extern "C" fmmb_status fmmb_perturb(fmmb_handle_t h, double* x, int64_t n, uint64_t seed,
                                    uint64_t step, double scale, void* stream) {
  FMMB_GUARD(h);
  if (n < 0 || (n > 0 && !x)) return FMMB_ERR_ARG;
  cudaSetDevice(h->device);
  if (n == 0) return FMMB_OK;
  const int64_t pairs = (n + 1) / 2;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((pairs + 255) / 256,
                                                               (int64_t)h->num_sms * 16));
  fmmb::k_perturb<<<grid, 256, 0, (cudaStream_t)stream>>>(x, n, seed, step, scale);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fmmb_fail(h, FMMB_ERR_CUDA, "perturb: %s", cudaGetErrorString(e));
  return FMMB_OK;
}
