// Shared device helpers for libfmmb200: Morton bit dilation, the compiled
// backend's exact f64 quantisation, decoupled-lookback tile states and warp
// primitives.  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fmmb200.h"

namespace fmmb {

constexpr int kMaxLevel = FMMB_MAX_LEVEL;
constexpr uint64_t kDilated = 0x1249249249249249ull;  // bit 3k set, k < 21

// ---------------------------------------------------------------- Morton --
// Insert two zero bits between the low 21 bits of v (digit = iz*4+iy*2+ix,
// coarsest level most significant: morton.py:1-7, _pykernels.py:22-30).
__host__ __device__ __forceinline__ uint64_t dilate3(uint64_t v) {
  v &= 0x1FFFFFull;
  v = (v | (v << 32)) & 0x001F00000000FFFFull;
  v = (v | (v << 16)) & 0x001F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & kDilated;
  return v;
}

// Inverse of dilate3 on the bits at positions 3k (_pykernels.py:33-40).
__host__ __device__ __forceinline__ uint64_t undilate3(uint64_t v) {
  v &= kDilated;
  v = (v | (v >> 2)) & 0x10C30C30C30C30C3ull;
  v = (v | (v >> 4)) & 0x100F00F00F00F00Full;
  v = (v | (v >> 8)) & 0x001F0000FF0000FFull;
  v = (v | (v >> 16)) & 0x001F00000000FFFFull;
  v = (v | (v >> 32)) & 0x1FFFFFull;
  return v;
}

__host__ __device__ __forceinline__ uint64_t morton3(uint64_t ix, uint64_t iy,
                                                     uint64_t iz) {
  return dilate3(ix) | (dilate3(iy) << 1) | (dilate3(iz) << 2);
}

// (long long)v as compiled by gcc for x86-64 (cvttsd2si): truncation toward
// zero, and the "integer indefinite" 0x8000000000000000 for NaN and for
// values outside the int64 range.  The compiled backend's encode_points
// (_ckernels.pyx:97-99) has exactly these semantics.
__device__ __forceinline__ long long trunc_ll_x86(double v) {
  if (v >= -9223372036854775808.0 && v < 9223372036854775808.0)
    return (long long)v;
  return (long long)0x8000000000000000ull;
}

// One coordinate of encode_points: `(long long)(x * 2^L)` clamped above at
// 2^L-1 (no lower clamp), _ckernels.pyx:96-102.  x * 2^L is exact in f64.
__device__ __forceinline__ uint64_t quantize_axis(double x, int level) {
  const double grid = (double)(1ll << level);
  long long i = trunc_ll_x86(__dmul_rn(x, grid));
  const long long hi = (1ll << level) - 1;
  if (i > hi) i = hi;
  return (uint64_t)i;
}

__device__ __forceinline__ uint64_t encode_point(double x, double y, double z,
                                                 int level) {
  return morton3(quantize_axis(x, level), quantize_axis(y, level),
                 quantize_axis(z, level));
}

// 10-bit dilation in 32-bit arithmetic (levels <= 10: 3L <= 30 key bits).
__device__ __forceinline__ uint32_t dilate3_10(uint32_t v) {
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// encode_point for level <= 10 with a 32-bit fast path: when every scaled
// coordinate t = x * 2^L lies in [0, 2^L) (the unit cube minus its upper
// faces) truncation is a plain conversion; anything else (x = 1.0 clamps,
// negative / NaN / huge inputs) takes the exact reference path.  Returns the
// same 64-bit key as encode_point.
__device__ __forceinline__ uint64_t encode_point_narrow(double x, double y, double z,
                                                        int level, double grid) {
  const double tx = __dmul_rn(x, grid), ty = __dmul_rn(y, grid), tz = __dmul_rn(z, grid);
  if (tx >= 0.0 && tx < grid && ty >= 0.0 && ty < grid && tz >= 0.0 && tz < grid) {
    // floor(t) for 0 <= t < 2^31 without the (XU-pipe) F2I conversion:
    // 2^52 + t rounded toward zero is 2^52 + floor(t); its low word is floor(t)
    constexpr double kMagic = 4503599627370496.0;  // 2^52
    const uint32_t ix = (uint32_t)__double2loint(__dadd_rz(tx, kMagic)),
                   iy = (uint32_t)__double2loint(__dadd_rz(ty, kMagic)),
                   iz = (uint32_t)__double2loint(__dadd_rz(tz, kMagic));
    return dilate3_10(ix) | (dilate3_10(iy) << 1) | (dilate3_10(iz) << 2);
  }
  return encode_point(x, y, z, level);
}

// level-generic entry: NARROW selects the 32-bit fast path (level <= 10)
template <bool NARROW>
__device__ __forceinline__ uint64_t encode_any(double x, double y, double z, int level,
                                               double grid) {
  if (NARROW) return encode_point_narrow(x, y, z, level, grid);
  return encode_point(x, y, z, level);
}

// ------------------------------------------------- decoupled look-back ----
// 64-bit tile state: [63:62] status, [61:0] value (Merrill & Garland 2016).
constexpr uint64_t kStInvalid = 0ull;
constexpr uint64_t kStAggregate = 1ull << 62;
constexpr uint64_t kStInclusive = 2ull << 62;
constexpr uint64_t kStMask = 3ull << 62;
constexpr uint64_t kStValue = ~kStMask;

__device__ __forceinline__ void st_state(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v)
               : "memory");
}
__device__ __forceinline__ uint64_t ld_state(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p)
               : "memory");
  return v;
}

// Sum of tile aggregates before `tile` for one counter (`stride` apart per
// tile), stopping at the first inclusive prefix or at `first_tile`.
__device__ __forceinline__ uint64_t lookback(const uint64_t* states,
                                             int64_t tile, int64_t first_tile,
                                             int64_t stride) {
  uint64_t excl = 0;
  int64_t t = tile - 1;
  while (t >= first_tile) {
    uint64_t s;
    do {
      s = ld_state(states + t * stride);
    } while ((s & kStMask) == kStInvalid);
    excl += s & kStValue;
    if ((s & kStMask) == kStInclusive) break;
    --t;
  }
  return excl;
}

// Same look-back run by one whole warp: lane i polls tile t-1-i of a 32-tile
// window, the window stops at its nearest inclusive prefix, else every
// aggregate is added and the window slides 32 tiles back.  One round trip
// per 32 predecessors instead of one per predecessor.  All lanes return the
// same value.
__device__ __forceinline__ uint64_t lookback_warp(const uint64_t* states,
                                                  int64_t tile, int64_t first_tile,
                                                  int64_t stride) {
  const int lane = (int)(threadIdx.x & 31u);
  uint64_t excl = 0;
  for (int64_t top = tile - 1; top >= first_tile; top -= 32) {
    const int64_t t = top - lane;
    uint64_t s = kStInclusive;  // before the segment: inclusive 0
    if (t >= first_tile) {
      do {
        s = ld_state(states + t * stride);
      } while ((s & kStMask) == kStInvalid);
    }
    const unsigned inc = __ballot_sync(0xffffffffu, (s & kStMask) == kStInclusive);
    const int stop = inc ? __ffs(inc) - 1 : 31;
    uint64_t v = lane <= stop ? (s & kStValue) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (inc) break;
  }
  return excl;
}

// --------------------------------------------------------------- warps ----
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_excl_scan(T v, T& total) {
  const unsigned lane = lane_id();
  T x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= (unsigned)d) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) {
  return (a + b - 1) / b;
}
__host__ __device__ __forceinline__ int64_t round_up(int64_t a, int64_t b) {
  return ceil_div(a, b) * b;
}

}  // namespace fmmb
