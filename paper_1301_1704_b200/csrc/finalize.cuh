// K3+K4: permuted gather of the sorted point sets fused with box-boundary
// detection and bookmark/non-empty compaction; K5: the occupancy-bitmap
// pyramid, its popcount rank directory and the per-level box directory.
//
// Reference: pseudosort.reorder (pseudosort.py:105-135) and build_bookmarks
// (:68-78) produce points/charges/permutation/boxes and (bookmarks,
// non_empty_index) from a dense 8^L histogram; lists.build_level_directory
// (lists.py:108-116) derives the coarse levels by np.unique(k >> 3).  Here
// the bookmarks come from head flags over the sorted keys (no dense grid), and
// every coarser level is a bitmap whose bit p = OR of byte p of the finer
// bitmap (the 8 children of box p are exactly that byte).
#pragma once
#include "common.cuh"

namespace fmmb {

constexpr int kGThreads = 256;
constexpr int kGWarps = kGThreads / 32;
constexpr int kGItems = 8;
constexpr int kGTile = kGThreads * kGItems;  // 2048 sorted positions

__host__ inline size_t gather_smem_bytes() {
  return (size_t)kGTile * 3 * sizeof(double) + (kGItems * kGWarps + 16) * 8;
}

// Sorted (key, idx) -> reference-layout outputs.  Combined layout: positions
// [0, n) are sources, [n, n+m) receivers.  Boxes get combined ranks j:
// ne_out[j] = Morton key; bm_out[j + set] = first sorted position within the
// set, so bm_out = [src bookmarks (K_s+1) | recv bookmarks (K_r+1)] once the
// two terminal entries (n, m) are written.  Heads also set the level-L
// occupancy bit of their set.
template <typename KeyT>
__global__ void __launch_bounds__(kGThreads)
    k_gather(const KeyT* __restrict__ skeys, const uint32_t* __restrict__ svals,
             int64_t n, int64_t m, int level, const double* __restrict__ src,
             const double* __restrict__ q, const double* __restrict__ recv,
             double* __restrict__ pts_out, double* __restrict__ q_out,
             int64_t* __restrict__ perm_out, uint64_t* __restrict__ boxes_out,
             uint64_t* __restrict__ ne_out, int64_t* __restrict__ bm_out,
             unsigned long long* __restrict__ bmp_src,
             unsigned long long* __restrict__ bmp_recv,
             uint64_t* __restrict__ states, uint32_t* __restrict__ tile_counter,
             int64_t* __restrict__ kinfo, const int64_t* __restrict__ gid_src,
             const int64_t* __restrict__ gid_recv) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_pts = reinterpret_cast<double*>(smem);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_pts + kGTile * 3);  // [items][warps]
  int64_t* s_misc = reinterpret_cast<int64_t*>(s_cnt + kGItems * kGWarps);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_misc[0] = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const int64_t tile = s_misc[0];
  const int64_t tbase = tile * kGTile;
  const int64_t total = n + m;
  const int sbits = 3 * level;
  const uint64_t kmask = (1ull << sbits) - 1;

  KeyT key[kGItems];
  unsigned heads[kGItems];
#pragma unroll
  for (int k = 0; k < kGItems; ++k) {
    const int64_t p = tbase + k * kGThreads + tid;
    bool head = false;
    if (p < total) {
      key[k] = skeys[p];
      head = (p == 0) || (skeys[p - 1] != key[k]);
    }
    heads[k] = __ballot_sync(0xffffffffu, head);
    if (lane == 0) s_cnt[k * kGWarps + warp] = __popc(heads[k]);
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan over (item, warp) in position order
    const uint32_t a = s_cnt[2 * lane], b = s_cnt[2 * lane + 1];
    uint32_t tot;
    const uint32_t x = warp_excl_scan(a + b, tot);
    s_cnt[2 * lane] = x;
    s_cnt[2 * lane + 1] = x + a;
    if (lane == 0) {
      uint64_t* st = states + tile;
      uint64_t excl = 0;
      if (tile == 0) {
        st_state(st, kStInclusive | tot);
      } else {
        st_state(st, kStAggregate | tot);
        excl = lookback(states, tile, 0, 1);
        st_state(st, kStInclusive | (excl + tot));
      }
      s_misc[1] = (int64_t)excl;
    }
  }
  __syncthreads();
  const int64_t toff = s_misc[1];

#pragma unroll
  for (int k = 0; k < kGItems; ++k) {
    const int64_t p = tbase + k * kGThreads + tid;
    if (p >= total) continue;
    const uint64_t ck = (uint64_t)key[k];
    const int set = (int)(ck >> sbits);
    const uint64_t mk = ck & kmask;
    const uint32_t idx = svals[p];
    const int64_t orig = set ? (int64_t)idx - n : (int64_t)idx;
    const double* row = set ? recv + 3 * orig : src + 3 * orig;
    const int r = k * kGThreads + tid;
    s_pts[3 * r + 0] = __ldg(row);
    s_pts[3 * r + 1] = __ldg(row + 1);
    s_pts[3 * r + 2] = __ldg(row + 2);
    perm_out[p] = set ? (gid_recv ? gid_recv[orig] : orig) : (gid_src ? gid_src[orig] : orig);
    boxes_out[p] = mk;
    if (!set && q) q_out[p] = __ldg(q + orig);
    // inclusive count of heads up to p = (combined rank of p's box) + 1
    const int64_t incl = toff + s_cnt[k * kGWarps + warp] +
                         __popc(heads[k] & (lanemask_lt() | (1u << lane)));
    if ((heads[k] >> lane) & 1u) {
      const int64_t j = incl - 1;
      ne_out[j] = mk;
      bm_out[j + set] = p - (set ? n : 0);
      unsigned long long* bm = set ? bmp_recv : bmp_src;
      if (bm) atomicOr(bm + (mk >> 6), 1ull << (mk & 63));
    }
    if (p == n - 1) {  // last source: terminal src bookmark (and empty recv)
      kinfo[0] = incl;
      bm_out[incl] = n;
      if (m == 0) bm_out[incl + 1] = 0;
    }
    if (p == total - 1 && m > 0) {
      kinfo[1] = incl;
      bm_out[incl + 1] = m;
      if (n == 0) { bm_out[0] = 0; kinfo[0] = 0; }
    }
  }
  __syncthreads();
  // coalesced 16-byte write-out of the staged point rows
  const int64_t left = total - tbase;
  const int nrows = left < kGTile ? (int)left : kGTile;
  const int ndbl = nrows * 3;
  double2* dst2 = reinterpret_cast<double2*>(pts_out + tbase * 3);
  const double2* s2 = reinterpret_cast<const double2*>(s_pts);
  for (int i = tid; i < ndbl / 2; i += kGThreads) dst2[i] = s2[i];
  if ((ndbl & 1) && tid == 0) pts_out[tbase * 3 + ndbl - 1] = s_pts[ndbl - 1];
}

// bit p of the result = (byte p of the 64-bit word x) != 0, for p < 8
__device__ __forceinline__ uint32_t nonzero_bytes(uint64_t x) {
  uint64_t t = (x & 0x7F7F7F7F7F7F7F7Full) + 0x7F7F7F7F7F7F7F7Full;
  t = (t | x) & 0x8080808080808080ull;
  return (uint32_t)(((t >> 7) * 0x0102040810204080ull) >> 56);
}

// One pyramid step for both sets: coarse word w = OR-reduction of the 64
// bytes in fine words [8w, 8w+8).  Fine segments are zero-padded to >= 8 words.
__global__ void k_pyramid(const uint64_t* __restrict__ fine0,
                          uint64_t* __restrict__ coarse0,
                          const uint64_t* __restrict__ fine1,
                          uint64_t* __restrict__ coarse1, int64_t ncoarse) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * ncoarse) return;
  const bool second = i >= ncoarse;
  const int64_t w = second ? i - ncoarse : i;
  const uint64_t* f = (second ? fine1 : fine0) + 8 * w;
  uint64_t out = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) out |= (uint64_t)nonzero_bytes(__ldg(f + b)) << (8 * b);
  (second ? coarse1 : coarse0)[w] = out;
}

constexpr int kMaxSegs = 2 * (kMaxLevel + 1);

struct PyramidTail {  // the small levels, reduced by one CTA
  uint64_t* lvl[2][kMaxLevel + 1];
  int64_t nwords[kMaxLevel + 1];
  int from_level;  // reduce from_level -> from_level-1 -> ... -> 0
};

__global__ void __launch_bounds__(1024) k_pyramid_tail(PyramidTail p) {
  for (int l = p.from_level; l >= 1; --l) {
    const int64_t nc = p.nwords[l - 1];
    for (int64_t i = threadIdx.x; i < 2 * nc; i += blockDim.x) {
      const int s = i >= nc;
      const int64_t w = s ? i - nc : i;
      const uint64_t* f = p.lvl[s][l] + 8 * w;
      uint64_t out = 0;
      for (int b = 0; b < 8; ++b) out |= (uint64_t)nonzero_bytes(f[b]) << (8 * b);
      p.lvl[s][l - 1][w] = out;
    }
    __syncthreads();
  }
}

// Rank directory: exclusive popcount scan of every (set, level) bitmap
// segment (segments start on tile boundaries, so a tile never spans two),
// the per-segment totals K_{set,l}, and the ascending box keys of each level
// (the reference LevelDirectory arrays, lists.py:108-116).
constexpr int kRThreads = 256;
constexpr int kRWordsPerThread = 4;
constexpr int kRTileWords = kRThreads * kRWordsPerThread;  // 1024 words

struct RankParams {
  const uint64_t* bmp;
  uint32_t* dir;
  uint64_t* states;
  uint32_t* tile_counter;
  int64_t* totals;  // [kMaxSegs]
  int nseg;
  int64_t word_off[kMaxSegs];
  int64_t nwords[kMaxSegs];
  int64_t tile_off[kMaxSegs + 1];
  uint64_t* keys_out[kMaxSegs];  // may be null
};

__global__ void __launch_bounds__(kRThreads) k_rank(const __grid_constant__ RankParams p) {
  __shared__ int64_t s_tile, s_excl;
  __shared__ uint32_t s_tmp[kRThreads / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(p.tile_counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  if (tile >= p.tile_off[p.nseg]) return;
  int seg = 0;
  while (p.tile_off[seg + 1] <= tile) ++seg;
  const int64_t first_tile = p.tile_off[seg];
  const int64_t wl0 = (tile - first_tile) * kRTileWords + tid * kRWordsPerThread;
  const uint64_t* words = p.bmp + p.word_off[seg];
  uint64_t w[kRWordsPerThread];
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < kRWordsPerThread; ++i) {
    w[i] = words[wl0 + i];  // padding words are zero
    c += __popcll(w[i]);
  }
  uint32_t wt;
  const uint32_t x = warp_excl_scan(c, wt);
  if (lane == 0) s_tmp[warp] = wt;
  __syncthreads();
  uint32_t off = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < kRThreads / 32; ++i) {
    off += i < warp ? s_tmp[i] : 0u;
    tot += s_tmp[i];
  }
  if (warp == 0) {
    uint64_t* st = p.states + tile;
    uint64_t excl = 0;
    if (tile == first_tile) {
      if (lane == 0) st_state(st, kStInclusive | tot);
    } else {
      if (lane == 0) st_state(st, kStAggregate | tot);
      excl = lookback_warp(p.states, tile, first_tile, 1);
      if (lane == 0) st_state(st, kStInclusive | (excl + tot));
    }
    if (lane == 0) {
      s_excl = (int64_t)excl;
      if (tile == p.tile_off[seg + 1] - 1) p.totals[seg] = (int64_t)(excl + tot);
    }
  }
  __syncthreads();
  uint64_t r = (uint64_t)s_excl + x + off;
  uint32_t* dir = p.dir + p.word_off[seg];
  uint64_t* keys = p.keys_out[seg];
  uint64_t rr[kRWordsPerThread];
#pragma unroll
  for (int i = 0; i < kRWordsPerThread; ++i) {
    const int64_t wl = wl0 + i;
    rr[i] = r;
    if (wl < p.nwords[seg]) dir[wl] = (uint32_t)r;
    r += __popcll(w[i]);
  }
  if (keys) {
    // box keys, warp-cooperative: one bitmap word at a time, lane = bits
    // lane and lane + 32, so a word's keys leave as one coalesced store
    // (per-thread bit loops wrote 32 scattered streams of up to 256 keys)
    const uint64_t below_lo = (1ull << lane) - 1ull;
    const uint64_t below_hi = lane == 31 ? 0x7FFFFFFFFFFFFFFFull : (1ull << (lane + 32)) - 1ull;
    for (int srcl = 0; srcl < 32; ++srcl) {
#pragma unroll
      for (int i = 0; i < kRWordsPerThread; ++i) {
        const uint64_t b = __shfl_sync(0xffffffffu, w[i], srcl);
        if (b == 0) continue;  // warp-uniform
        const uint64_t r0 = __shfl_sync(0xffffffffu, rr[i], srcl);
        const int64_t wl = wl0 + (int64_t)(srcl - lane) * kRWordsPerThread + i;
        if ((b >> lane) & 1ull) keys[r0 + __popcll(b & below_lo)] = (uint64_t)wl * 64 + lane;
        if ((b >> (lane + 32)) & 1ull)
          keys[r0 + __popcll(b & below_hi)] = (uint64_t)wl * 64 + lane + 32;
      }
    }
  }
}

}  // namespace fmmb
