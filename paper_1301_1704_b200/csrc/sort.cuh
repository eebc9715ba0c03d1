// K1 encode + K2 stable LSD radix sort (Onesweep) of (combined key, index).
//
// Replaces the reference pseudo-sort histogram + rank + reorder
// (pseudosort.py:41-65,105-135; _ckernels.pyx:85-119).  The reference's
// contract is "within-box order = input order" (`assign_box_ranks`, a
// sequential per-box counter), i.e. the permutation equals
// np.argsort(keys, kind="stable") (tests/test_pseudosort.py:94-104).  A
// stable LSD radix sort over (key, original index) pairs produces exactly
// that order without the reference's dense 8^L histogram.
//
// Sources and receivers are sorted in ONE pass set: receiver keys carry a set
// bit above the 3L Morton bits, so the sorted array is [src sorted | recv
// sorted] and both sets share every launch.
#pragma once
#include "common.cuh"

namespace fmmb {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 pairs per tile
constexpr int kRadixBits = 8;
constexpr int kBins = 1 << kRadixBits;
constexpr int kMaxPasses = 8;  // 3*20+1 = 61 key bits

__host__ __device__ inline int sort_key_bits(int level) { return 3 * level + 1; }
__host__ __device__ inline int sort_passes(int level) {
  return (sort_key_bits(level) + kRadixBits - 1) / kRadixBits;
}

// Block-wide exclusive scan of one value per thread (kSortThreads threads).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_tmp,
                                                    uint32_t* total = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t wt;
  uint32_t x = warp_excl_scan(v, wt);
  if (lane == 0) s_tmp[warp] = wt;
  __syncthreads();
  uint32_t off = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) {
    uint32_t t = s_tmp[w];
    off += (w < warp) ? t : 0u;
    all += t;
  }
  __syncthreads();
  if (total) *total = all;
  return x + off;
}

// K1: quantise + interleave every point of [src | recv], write the combined
// key (Morton key | set bit << 3L) and accumulate the digit histograms of all
// radix passes (Onesweep's single upsweep).  Flags keys outside the level
// grid (reference UB: negative coordinates index its histogram out of
// bounds, _ckernels.pyx:115-118).
template <typename KeyT>
__global__ void __launch_bounds__(kSortThreads)
    k_encode_hist(const double* __restrict__ src, int64_t n,
                  const double* __restrict__ recv, int64_t m, int level,
                  int npass, KeyT* __restrict__ keys,
                  uint32_t* __restrict__ hist, uint32_t* __restrict__ err) {
  __shared__ uint32_t sh[kMaxPasses * kBins];
  for (int i = threadIdx.x; i < npass * kBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t total = n + m;
  const int sbits = 3 * level;
  const uint64_t lim = 1ull << sbits;
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += stride) {
    const bool is_recv = i >= n;
    const double* p = is_recv ? recv + 3 * (i - n) : src + 3 * i;
    const double x = __ldg(p), y = __ldg(p + 1), z = __ldg(p + 2);
    const uint64_t key = encode_point(x, y, z, level);
    bad |= key >= lim;
    const uint64_t ck = (key & (lim - 1)) | ((uint64_t)is_recv << sbits);
    keys[i] = (KeyT)ck;
    for (int ps = 0; ps < npass; ++ps)
      atomicAdd(&sh[ps * kBins + (int)((ck >> (kRadixBits * ps)) & (kBins - 1))], 1u);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < npass * kBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// Digit histograms of precomputed u64 keys (plugin-level sorts): writes the
// keys narrowed to KeyT and flags keys >= limit.
template <typename KeyT>
__global__ void __launch_bounds__(kSortThreads)
    k_keys_hist(const uint64_t* __restrict__ kin, int64_t n, uint64_t limit, int npass,
                KeyT* __restrict__ keys, uint32_t* __restrict__ hist,
                uint32_t* __restrict__ err) {
  __shared__ uint32_t sh[kMaxPasses * kBins];
  for (int i = threadIdx.x; i < npass * kBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = kin[i];
    bad |= k >= limit;
    keys[i] = (KeyT)k;
    for (int ps = 0; ps < npass; ++ps)
      atomicAdd(&sh[ps * kBins + (int)((k >> (kRadixBits * ps)) & (kBins - 1))], 1u);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < npass * kBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__host__ inline size_t onesweep_smem_bytes(size_t key_bytes) {
  return (size_t)kSortTile * (key_bytes + 4) +
         (size_t)(kSortWarps * kBins + 3 * kBins + 16) * 4;
}

// K2: one Onesweep digit pass (Adinets & Merrill 2022).  Each CTA takes the
// next tile id (atomic ticket => tiles start in order, look-back never waits
// on an unscheduled tile), ranks its 4096 pairs stably per digit with warp
// match-any + per-warp counters, publishes its per-digit counts, resolves its
// global per-digit offset by decoupled look-back, and scatters the pairs in
// digit-grouped runs (coalesced) from shared memory.
template <typename KeyT, bool FIRST>
__global__ void __launch_bounds__(kSortThreads)
    k_onesweep(const KeyT* __restrict__ kin, const uint32_t* __restrict__ vin,
               KeyT* __restrict__ kout, uint32_t* __restrict__ vout,
               int64_t total, int shift, const uint32_t* __restrict__ hist,
               uint64_t* __restrict__ states,
               uint32_t* __restrict__ tile_counter) {
  extern __shared__ __align__(16) unsigned char smem[];
  KeyT* s_keys = reinterpret_cast<KeyT*>(smem);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + kSortTile);
  uint32_t* s_whist = s_vals + kSortTile;  // [warps][bins]
  uint32_t* s_bin = s_whist + kSortWarps * kBins;
  uint32_t* s_texc = s_bin + kBins;
  uint32_t* s_gb = s_texc + kBins;
  uint32_t* s_misc = s_gb + kBins;  // [0]=tile, [8..15] scan scratch

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_misc[0] = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < kSortWarps * kBins; i += kSortThreads) s_whist[i] = 0;
  // global start of each digit bin = exclusive scan of this pass's histogram
  s_bin[tid] = block_excl_scan(hist[tid], s_misc + 8);  // syncs inside
  const int64_t tile = s_misc[0];
  const int64_t tbase = tile * kSortTile;
  const int64_t wbase = tbase + (int64_t)warp * (32 * kSortItems);

  KeyT keys[kSortItems];
  uint32_t vals[kSortItems];
  uint32_t rank[kSortItems];
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const int64_t pos = wbase + k * 32 + lane;
    const bool ok = pos < total;
    keys[k] = ok ? kin[pos] : (KeyT)0;
    vals[k] = FIRST ? (uint32_t)pos : (ok ? vin[pos] : 0u);
  }
  // stable in-warp ranking: items visited in element order (k-major, lane)
  uint32_t* wh = s_whist + warp * kBins;
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const int64_t pos = wbase + k * 32 + lane;
    const int d = pos < total ? (int)((keys[k] >> shift) & (kBins - 1)) : kBins;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(peers) - 1;
    uint32_t before = 0;
    if (lane == leader && d < kBins) {
      before = wh[d];
      wh[d] = before + __popc(peers);
    }
    before = __shfl_sync(0xffffffffu, before, leader);
    rank[k] = before + __popc(peers & lanemask_lt());
    __syncwarp();
  }
  __syncthreads();
  // thread = digit bin: tile count and per-warp exclusive offsets
  uint32_t c = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) {
    const uint32_t x = s_whist[w * kBins + tid];
    s_whist[w * kBins + tid] = c;
    c += x;
  }
  uint64_t* st = states + tile * kBins + tid;
  st_state(st, (tile == 0 ? kStInclusive : kStAggregate) | (uint64_t)c);
  s_texc[tid] = block_excl_scan(c, s_misc + 8);
  uint64_t excl = 0;
  if (tile > 0) {
    excl = lookback(states + tid, tile, 0, kBins);
    st_state(st, kStInclusive | (excl + c));
  }
  s_gb[tid] = s_bin[tid] + (uint32_t)excl - s_texc[tid];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const int64_t pos = wbase + k * 32 + lane;
    if (pos < total) {
      const int d = (int)((keys[k] >> shift) & (kBins - 1));
      const uint32_t lp = s_texc[d] + s_whist[warp * kBins + d] + rank[k];
      s_keys[lp] = keys[k];
      s_vals[lp] = vals[k];
    }
  }
  __syncthreads();
  const int64_t left = total - tbase;
  const int nvalid = left < kSortTile ? (int)left : kSortTile;
  for (int j = tid; j < nvalid; j += kSortThreads) {
    const KeyT key = s_keys[j];
    const int d = (int)((key >> shift) & (kBins - 1));
    const uint32_t dst = s_gb[d] + (uint32_t)j;
    kout[dst] = key;
    vout[dst] = s_vals[j];
  }
}

}  // namespace fmmb
