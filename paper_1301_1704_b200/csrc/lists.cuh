// K6/K7: E2 neighbour lists and E4 interaction (translation-stencil) lists.
//
// Reference: adjacent_segments (_ckernels.pyx:140-202) and stencil_segments
// (_ckernels.pyx:205-287), called by build_neighbor_table (lists.py:69-77)
// and build_translation_stencils (lists.py:119-130).  Both enumerate, per
// receiver box r at level l, the children of the parent's 3x3x3 window in
// ascending Morton order (the parent window sorted, children 8p..8p+7
// ascending), keeping occupied source boxes; E2 keeps the ones in r's own
// window (|d|<=1 per axis), E4 the others.  Both lists therefore come out of
// ONE enumeration over the 6x6x6 block of children of the parent window.
//
// One warp per receiver PARENT box P (level l-1): lanes 0..26 take the 27
// window offsets of P, Morton keys are sorted across lanes (bitonic), and a
// lane's 8 candidate children are one byte of the level-l source occupancy
// bitmap; their ranks come from the popcount rank directory (O(1), no
// search).  P's child receivers are one byte of the receiver bitmap.
// count pass -> segmented scan (CSR bookmarks) -> write pass staged in shared
// memory and streamed out with coalesced stores.
#pragma once
#include "common.cuh"

namespace fmmb {

constexpr int kLThreads = 256;
constexpr int kLWarps = kLThreads / 32;
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048 counts

// Segment ids of the count/bookmark arrays: 0 = E2 at max level, l = E4 at l.
struct ListsParams {
  int level;                 // L
  const int64_t* ktot;       // [2*(L+1)]: K_{set,l} at index set*(L+1)+l
  const uint64_t* bmp;       // bitmaps, both sets
  const uint32_t* dir;       // rank directories, same layout
  int64_t bmp_off[2][kMaxLevel + 1];
  const uint64_t* rkeys[kMaxLevel + 1];  // receiver box keys per level < L
  uint32_t* counts;          // padded segments (count pass output)
  int64_t* bm[kMaxLevel + 1];            // bookmark arrays per segment
  int64_t* ranks_out[kMaxLevel + 1];     // write pass: [0]=E2 list, [l]=E4 ranks
  int16_t* codes_out[kMaxLevel + 1];     // [l]=E4 codes
};

// Per-level work and segment layout, recomputed per block from the device
// totals (<= 21 levels).
struct ListsLayout {
  int lmin;                     // first level with work
  int64_t work_off[kMaxLevel + 2];  // prefix of receiver-parent counts
  int64_t seg_len[kMaxLevel + 1];
  int64_t seg_off[kMaxLevel + 2];
};

__device__ __forceinline__ int lists_lmin(int L) { return L >= 2 ? 2 : L; }

__device__ inline void lists_layout(const ListsParams& p, ListsLayout& lay) {
  const int L = p.level;
  const int stride = L + 1;
  lay.lmin = lists_lmin(L);
  int64_t w = 0;
  for (int l = 0; l <= kMaxLevel + 1; ++l) lay.work_off[l] = 0;
  for (int l = 0; l <= L; ++l) {
    lay.work_off[l] = w;
    if (l >= lay.lmin) w += (l == 0) ? p.ktot[stride + 0] : p.ktot[stride + l - 1];
  }
  lay.work_off[L + 1] = w;
  int64_t off = 0;
  for (int s = 0; s <= kMaxLevel; ++s) {
    int64_t len = 0;
    if (s == 0) len = p.ktot[stride + L] + 1;
    else if (s >= 2 && s <= L) len = p.ktot[stride + s] + 1;
    lay.seg_len[s] = len;
    lay.seg_off[s] = off;
    off += round_up(len, kScanTile);
  }
  lay.seg_off[kMaxLevel + 1] = off;
}

__device__ __forceinline__ void children_of(const uint64_t* bmp,
                                            const uint32_t* dir, uint64_t p,
                                            uint32_t& mask, uint32_t& first) {
  const uint64_t w = __ldg(bmp + (p >> 3));
  const int sh = (int)(p & 7) * 8;
  mask = (uint32_t)(w >> sh) & 0xFFu;
  first = __ldg(dir + (p >> 3)) + (uint32_t)__popcll(w & ((1ull << sh) - 1ull));
}

// children c of neighbour-parent offset o that lie in child-receiver cr's own
// 3x3x3 window: per axis, offset 0 keeps all, -1 keeps c_a=1 iff cr_a=0,
// +1 keeps c_a=0 iff cr_a=1.
__device__ __forceinline__ uint32_t near_mask(int ox, int oy, int oz, int cr) {
  uint32_t mk = 0xFFu;
  const int o[3] = {ox, oy, oz};
  const uint32_t hi[3] = {0xAAu, 0xCCu, 0xF0u};  // children with bit a set
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int ca = (cr >> a) & 1;
    if (o[a] < 0) mk &= ca == 0 ? hi[a] : 0u;
    else if (o[a] > 0) mk &= ca == 1 ? (~hi[a] & 0xFFu) : 0u;
  }
  return mk;
}

template <bool WRITE>
__global__ void __launch_bounds__(kLThreads) k_lists(const __grid_constant__ ListsParams p) {
  __shared__ ListsLayout lay;
  __shared__ int64_t s_r4[kLWarps][192];
  __shared__ int16_t s_c4[kLWarps][192];
  __shared__ int64_t s_r2[kLWarps][32];
  if (threadIdx.x == 0) lists_layout(p, lay);
  __syncthreads();
  const int L = p.level;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwork = lay.work_off[L + 1];
  const int64_t gw0 = (int64_t)blockIdx.x * kLWarps + warp;
  const int64_t gstride = (int64_t)gridDim.x * kLWarps;
  const unsigned FULL = 0xffffffffu;

  for (int64_t gw = gw0; gw < nwork; gw += gstride) {
    int l = lay.lmin;
    while (lay.work_off[l + 1] <= gw) ++l;
    const int64_t j = gw - lay.work_off[l];
    if (l == 0) {  // max level 0: the root receiver sees the root source
      const int64_t ks = p.ktot[0];
      if (lane == 0) {
        if (!WRITE) p.counts[lay.seg_off[0]] = (uint32_t)ks;
        else if (ks) p.ranks_out[0][p.bm[0][0]] = 0;
      }
      continue;
    }
    const uint64_t P = p.rkeys[l - 1][j];
    const int64_t np = 1ll << (l - 1);
    const int64_t px = (int64_t)undilate3(P), py = (int64_t)undilate3(P >> 1),
                  pz = (int64_t)undilate3(P >> 2);
    int o = lane;
    uint64_t qk = ~0ull;
    if (lane < 27) {
      const int64_t qx = px + (lane % 3) - 1, qy = py + (lane / 3) % 3 - 1,
                    qz = pz + lane / 9 - 1;
      if (qx >= 0 && qx < np && qy >= 0 && qy < np && qz >= 0 && qz < np)
        qk = morton3((uint64_t)qx, (uint64_t)qy, (uint64_t)qz);
    }
    // bitonic sort of (qk, o) across the warp, ascending by lane
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (int d = k >> 1; d > 0; d >>= 1) {
        const uint64_t ok = __shfl_xor_sync(FULL, qk, d);
        const int oo = __shfl_xor_sync(FULL, o, d);
        const bool want_min = ((lane & d) == 0) == ((lane & k) == 0);
        if (want_min ? (ok < qk) : (ok > qk)) { qk = ok; o = oo; }
      }
    }
    uint32_t sm = 0, sfirst = 0;
    if (qk != ~0ull)
      children_of(p.bmp + p.bmp_off[0][l], p.dir + p.bmp_off[0][l], qk, sm, sfirst);
    uint32_t rm, rfirst;
    children_of(p.bmp + p.bmp_off[1][l], p.dir + p.bmp_off[1][l], P, rm, rfirst);
    const int ox = o % 3 - 1, oy = (o / 3) % 3 - 1, oz = o / 9 - 1;
    const bool do_e4 = l >= 2, do_e2 = l == L;
    uint32_t rbits = rm;
    while (rbits) {
      const int cr = __ffs(rbits) - 1;
      rbits &= rbits - 1;
      const int64_t rrank = rfirst + __popc(rm & ((1u << cr) - 1u));
      const uint32_t nm = near_mask(ox, oy, oz, cr);
      const uint32_t e4 = do_e4 ? (sm & ~nm) : 0u;
      const uint32_t e2 = do_e2 ? (sm & nm) : 0u;
      if (!WRITE) {
        const uint32_t c4 = __reduce_add_sync(FULL, (unsigned)__popc(e4));
        const uint32_t c2 = __reduce_add_sync(FULL, (unsigned)__popc(e2));
        if (lane == 0) {
          if (do_e4) p.counts[lay.seg_off[l] + rrank] = c4;
          if (do_e2) p.counts[lay.seg_off[0] + rrank] = c2;
        }
      } else {
        uint32_t t4, t2;
        uint32_t x4 = warp_excl_scan((uint32_t)__popc(e4), t4);
        uint32_t x2 = warp_excl_scan((uint32_t)__popc(e2), t2);
        const int cbase = (2 * ox - (cr & 1) + 3) + 7 * (2 * oy - ((cr >> 1) & 1) + 3) +
                          49 * (2 * oz - ((cr >> 2) & 1) + 3);
        uint32_t b = e4;
        while (b) {
          const int c = __ffs(b) - 1;
          b &= b - 1;
          s_r4[warp][x4] = (int64_t)(sfirst + __popc(sm & ((1u << c) - 1u)));
          s_c4[warp][x4] = (int16_t)(cbase + (c & 1) + 7 * ((c >> 1) & 1) + 49 * ((c >> 2) & 1));
          ++x4;
        }
        b = e2;
        while (b) {
          const int c = __ffs(b) - 1;
          b &= b - 1;
          s_r2[warp][x2++] = (int64_t)(sfirst + __popc(sm & ((1u << c) - 1u)));
        }
        __syncwarp();
        if (do_e4 && t4) {
          const int64_t row = p.bm[l][rrank];
          int64_t* dr = p.ranks_out[l] + row;
          int16_t* dc = p.codes_out[l] + row;
          for (uint32_t i = lane; i < t4; i += 32) {
            dr[i] = s_r4[warp][i];
            dc[i] = s_c4[warp][i];
          }
        }
        if (do_e2 && t2) {
          const int64_t row = p.bm[0][rrank];
          int64_t* dr = p.ranks_out[0] + row;
          for (uint32_t i = lane; i < t2; i += 32) dr[i] = s_r2[warp][i];
        }
        __syncwarp();
      }
    }
  }
}

// Segmented exclusive scan of the padded count array into the i64 bookmark
// arrays (one segment per list; segments start on tile boundaries and carry
// a trailing zero so bookmark[K] = segment total).  Single pass, decoupled
// look-back restarted at each segment's first tile.
__global__ void __launch_bounds__(kScanThreads) k_lists_scan(const __grid_constant__ ListsParams p,
                                                             uint64_t* __restrict__ states,
                                                             uint32_t* __restrict__ tile_counter,
                                                             int64_t* __restrict__ seg_totals) {
  __shared__ ListsLayout lay;
  __shared__ int64_t s_tile, s_excl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    lists_layout(p, lay);
    s_tile = atomicAdd(tile_counter, 1u);
  }
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t ntiles = lay.seg_off[kMaxLevel + 1] / kScanTile;
  if (tile >= ntiles) return;
  int seg = 0;
  while (lay.seg_off[seg + 1] / kScanTile <= tile) ++seg;
  const int64_t first_tile = lay.seg_off[seg] / kScanTile;
  const int64_t last_tile = lay.seg_off[seg + 1] / kScanTile - 1;
  const int64_t e0 = (tile - first_tile) * kScanTile + tid * kScanItems;
  const int64_t len = lay.seg_len[seg];
  const uint32_t* cnt = p.counts + lay.seg_off[seg];
  uint32_t v[kScanItems];
  uint64_t c = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t e = e0 + i;
    v[i] = (e < len - 1) ? cnt[e] : 0u;  // the trailing entry is the total
    c += v[i];
  }
  uint64_t wt;
  const uint64_t x = warp_excl_scan<uint64_t>(c, wt);
  __shared__ uint64_t s_w[kScanThreads / 32];
  if (lane == 0) s_w[warp] = wt;
  __syncthreads();
  uint64_t off = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < kScanThreads / 32; ++i) {
    off += i < warp ? s_w[i] : 0ull;
    tot += s_w[i];
  }
  if (tid == 0) {
    uint64_t* st = states + tile;
    uint64_t excl = 0;
    if (tile == first_tile) {
      st_state(st, kStInclusive | tot);
    } else {
      st_state(st, kStAggregate | tot);
      excl = lookback(states, tile, first_tile, 1);
      st_state(st, kStInclusive | (excl + tot));
    }
    s_excl = (int64_t)excl;
    if (tile == last_tile) seg_totals[seg] = (int64_t)(excl + tot);
  }
  __syncthreads();
  int64_t r = s_excl + (int64_t)(x + off);
  int64_t* bm = p.bm[seg];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t e = e0 + i;
    if (e < len) bm[e] = r;
    r += v[i];
  }
}

}  // namespace fmmb
