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

// One-time layout (per-level work and padded count segments) from the device
// totals; written to global memory for the count / scan / write kernels.
__global__ void k_lists_plan(const __grid_constant__ ListsParams p, ListsLayout* out) {
  if (threadIdx.x == 0) lists_layout(p, *out);
}

__device__ __forceinline__ void load_layout(const ListsLayout* g, ListsLayout& s) {
  const int words = sizeof(ListsLayout) / 4;
  for (int i = threadIdx.x; i < words; i += blockDim.x)
    reinterpret_cast<uint32_t*>(&s)[i] = reinterpret_cast<const uint32_t*>(g)[i];
}

// Neighbour window of P (level l-1) for lane o < 27 (o = ox+1 + 3(oy+1) +
// 9(oz+1)): the neighbour's Morton key by dilated-integer add/subtract on each
// axis (no de-interleave), or ~0 outside the level grid.
__device__ __forceinline__ uint64_t window_key(uint64_t P, int l, int o) {
  if (o >= 27) return ~0ull;
  const int bits = 3 * (l - 1);
  const uint64_t full = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
  uint64_t k = P;
  const int off[3] = {o % 3 - 1, (o / 3) % 3 - 1, o / 9 - 1};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const uint64_t m = (kDilated << a) & full;
    const uint64_t ka = k & m;
    if (off[a] > 0) {
      if (ka == m) return ~0ull;
      k = (((k | ~m) + 1ull) & m) | (k & ~m);
    } else if (off[a] < 0) {
      if (ka == 0) return ~0ull;
      k = ((ka - 1ull) & m) | (k & ~m);
    }
  }
  return k;
}

// NEAR[o] byte cr = children c of neighbour-parent offset o that lie in child
// receiver cr's own 3x3x3 window (per axis: offset 0 keeps all, -1 keeps
// c_a=1 iff cr_a=0, +1 keeps c_a=0 iff cr_a=1).
struct NearTable {
  uint64_t w[27];
  constexpr NearTable() : w() {
    for (int o = 0; o < 27; ++o) {
      const int off[3] = {o % 3 - 1, (o / 3) % 3 - 1, o / 9 - 1};
      uint64_t word = 0;
      for (int cr = 0; cr < 8; ++cr) {
        unsigned mk = 0;
        for (int c = 0; c < 8; ++c) {
          bool near = true;
          for (int a = 0; a < 3; ++a) {
            const int d = 2 * off[a] + ((c >> a) & 1) - ((cr >> a) & 1);
            near = near && d >= -1 && d <= 1;
          }
          if (near) mk |= 1u << c;
        }
        word |= (uint64_t)mk << (8 * cr);
      }
      w[o] = word;
    }
  }
};
__constant__ NearTable kNear = NearTable();

// per-byte popcount of a 64-bit word (each byte -> 0..8)
__device__ __forceinline__ uint64_t popc_bytes(uint64_t x) {
  x = x - ((x >> 1) & 0x5555555555555555ull);
  x = (x & 0x3333333333333333ull) + ((x >> 2) & 0x3333333333333333ull);
  return (x + (x >> 4)) & 0x0F0F0F0F0F0F0F0Full;
}

// Count pass: per child receiver r of P, |E4_l(r)| (and |E2(r)| at l == L).
// Lane = window slot; the near-children counts of all 8 child receivers come
// from one SWAR byte-popcount and two warp reductions.
__global__ void __launch_bounds__(kLThreads)
    k_lists_count(const __grid_constant__ ListsParams p, const ListsLayout* __restrict__ glay) {
  __shared__ ListsLayout lay;
  load_layout(glay, lay);
  __syncthreads();
  const int L = p.level;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwork = lay.work_off[L + 1];
  const int64_t gstride = (int64_t)gridDim.x * kLWarps;
  const unsigned FULL = 0xffffffffu;
  const uint64_t nearw = lane < 27 ? kNear.w[lane] : 0ull;
  for (int64_t gw = (int64_t)blockIdx.x * kLWarps + warp; gw < nwork; gw += gstride) {
    int l = lay.lmin;
    while (lay.work_off[l + 1] <= gw) ++l;
    const int64_t j = gw - lay.work_off[l];
    if (l == 0) {  // max level 0: the root receiver sees the root source
      if (lane == 0) p.counts[lay.seg_off[0]] = (uint32_t)p.ktot[0];
      continue;
    }
    const uint64_t P = __ldg(p.rkeys[l - 1] + j);
    const uint64_t qk = window_key(P, l, lane);
    uint32_t sm = 0, sfirst;
    if (qk != ~0ull)
      children_of(p.bmp + p.bmp_off[0][l], p.dir + p.bmp_off[0][l], qk, sm, sfirst);
    uint32_t rm, rfirst;
    children_of(p.bmp + p.bmp_off[1][l], p.dir + p.bmp_off[1][l], P, rm, rfirst);
    const uint64_t e2b = popc_bytes(((uint64_t)sm * 0x0101010101010101ull) & nearw);
    const uint32_t lo = __reduce_add_sync(FULL, (uint32_t)e2b);
    const uint32_t hi = __reduce_add_sync(FULL, (uint32_t)(e2b >> 32));
    const uint32_t all = __reduce_add_sync(FULL, (uint32_t)__popc(sm));
    if (lane < 8 && ((rm >> lane) & 1u)) {
      const uint32_t e2 = ((lane < 4 ? lo >> (8 * lane) : hi >> (8 * (lane - 4)))) & 0xFFu;
      const int64_t rrank = rfirst + __popc(rm & ((1u << lane) - 1u));
      if (l >= 2) p.counts[lay.seg_off[l] + rrank] = all - e2;
      if (l == L) p.counts[lay.seg_off[0] + rrank] = e2;
    }
  }
}

// Write pass.  Lanes hold the window neighbours sorted by Morton key; the
// 27x8 candidate children of a row are visited in output order as 7 chunks
// of 32 (lane = candidate: slot = 4*chunk + lane/8, child c = lane%8).  Every
// row-independent quantity of a chunk (occupancy, rank, code base, the near
// bit for each of the 8 child receivers) is computed once per P; a row is
// then one ballot-compaction per chunk with coalesced stores straight to HBM.
// The rows of P's child receivers are consecutive, so one bookmark read per P.
__device__ __forceinline__ unsigned ballot_full(unsigned pred) {
  unsigned b;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
               "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t}" : "=r"(b) : "r"(pred));
  return b;
}

// predicated stores (no branch around them)
__device__ __forceinline__ void st_rank_code(unsigned pred, int64_t* r, int64_t rank, int16_t* c,
                                             int code) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
      "@p st.global.s64 [%1], %2;\n\t@p st.global.s16 [%3], %4;\n\t}" ::"r"(pred),
      "l"(r), "l"(rank), "l"(c), "h"((short)code)
      : "memory");
}
__device__ __forceinline__ void st_rank(unsigned pred, int64_t* r, int64_t rank) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.global.s64 [%1], %2;\n\t}" ::
                   "r"(pred), "l"(r), "l"(rank)
               : "memory");
}

template <bool E4, bool E2>
__device__ __forceinline__ void write_rows(uint32_t rm, const uint32_t (&meta)[7],
                                           const uint32_t (&rank)[7], int64_t* __restrict__ r4,
                                           int16_t* __restrict__ c4, int64_t* __restrict__ r2) {
  const unsigned lt = lanemask_lt();
  uint32_t rbits = rm;
  while (rbits) {
    const int cr = __ffs(rbits) - 1;
    rbits &= rbits - 1;
    const int crw = (cr & 1) + 7 * ((cr >> 1) & 1) + 49 * ((cr >> 2) & 1);
    const int sh = 1 + cr;
#pragma unroll
    for (int ch = 0; ch < 7; ++ch) {
      const uint32_t m = meta[ch];
      const uint32_t nb = m >> sh;
      if (E4) {
        const unsigned v = m & ~nb & 1u;
        const unsigned b = ballot_full(v);
        const unsigned at = __popc(b & lt);
        st_rank_code(v, r4 + at, (int64_t)rank[ch], c4 + at, (int)(m >> 9) - crw);
        r4 += __popc(b);
        c4 += __popc(b);
      }
      if (E2) {
        const unsigned v = m & nb & 1u;
        const unsigned b = ballot_full(v);
        st_rank(v, r2 + __popc(b & lt), (int64_t)rank[ch]);
        r2 += __popc(b);
      }
    }
  }
}

__global__ void __launch_bounds__(kLThreads)
    k_lists_write(const __grid_constant__ ListsParams p, const ListsLayout* __restrict__ glay) {
  __shared__ ListsLayout lay;
  load_layout(glay, lay);
  __syncthreads();
  const int L = p.level;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwork = lay.work_off[L + 1];
  const int64_t gstride = (int64_t)gridDim.x * kLWarps;
  const unsigned FULL = 0xffffffffu;
  const int c = lane & 7;
  // code contribution of the candidate child c: (c_x + 7 c_y + 49 c_z) + 3*57
  const int cc = (c & 1) + 7 * ((c >> 1) & 1) + 49 * ((c >> 2) & 1) + 171;
  for (int64_t gw = (int64_t)blockIdx.x * kLWarps + warp; gw < nwork; gw += gstride) {
    int l = lay.lmin;
    while (lay.work_off[l + 1] <= gw) ++l;
    const int64_t j = gw - lay.work_off[l];
    if (l == 0) {
      if (lane == 0 && p.ktot[0]) p.ranks_out[0][p.bm[0][0]] = 0;
      continue;
    }
    const uint64_t P = __ldg(p.rkeys[l - 1] + j);
    uint64_t qk = window_key(P, l, lane);
    int o = lane;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (int d = k >> 1; d > 0; d >>= 1) {
        const uint64_t ok = __shfl_xor_sync(FULL, qk, d);
        const int oo = __shfl_xor_sync(FULL, o, d);
        const bool want_min = ((lane & d) == 0) == ((lane & k) == 0);
        if (want_min ? (ok < qk) : (ok > qk)) {
          qk = ok;
          o = oo;
        }
      }
    }
    uint32_t sm = 0, sfirst = 0;
    if (qk != ~0ull)
      children_of(p.bmp + p.bmp_off[0][l], p.dir + p.bmp_off[0][l], qk, sm, sfirst);
    uint32_t rm, rfirst;
    children_of(p.bmp + p.bmp_off[1][l], p.dir + p.bmp_off[1][l], P, rm, rfirst);
    // per chunk: meta = occ | near-over-cr (8 bits) << 1 | code base << 9
    const uint32_t slot_word = sm | ((uint32_t)(o < 27 ? o : 13) << 8);
    uint32_t meta[7], rank[7];
#pragma unroll
    for (int ch = 0; ch < 7; ++ch) {
      const int slot = 4 * ch + (lane >> 3);
      const uint32_t v = __shfl_sync(FULL, slot_word, slot);
      const uint32_t f = __shfl_sync(FULL, sfirst, slot);
      const uint32_t smk = v & 0xFFu;
      const int so = (int)(v >> 8);
      const uint64_t nw = kNear.w[so];
      uint32_t nearcr = 0;
#pragma unroll
      for (int cr = 0; cr < 8; ++cr) nearcr |= ((uint32_t)(nw >> (8 * cr + c)) & 1u) << cr;
      const int sx = so % 3 - 1, sy = (so / 3) % 3 - 1, sz = so / 9 - 1;
      const uint32_t code0 = (uint32_t)(2 * sx + 7 * 2 * sy + 49 * 2 * sz + cc);
      const bool occ = slot < 27 && ((smk >> c) & 1u);
      meta[ch] = (occ ? 1u : 0u) | (nearcr << 1) | (code0 << 9);
      rank[ch] = f + __popc(smk & ((1u << c) - 1u));
    }
    int64_t* r4 = p.ranks_out[l];
    int16_t* c4 = p.codes_out[l];
    int64_t* r2 = p.ranks_out[0];
    if (l == L) {
      const int64_t w2 = __ldg(p.bm[0] + rfirst);
      if (l >= 2) {
        const int64_t w4 = __ldg(p.bm[l] + rfirst);
        write_rows<true, true>(rm, meta, rank, r4 + w4, c4 + w4, r2 + w2);
      } else {
        write_rows<false, true>(rm, meta, rank, nullptr, nullptr, r2 + w2);
      }
    } else {
      const int64_t w4 = __ldg(p.bm[l] + rfirst);
      write_rows<true, false>(rm, meta, rank, r4 + w4, c4 + w4, nullptr);
    }
  }
}

// Segmented exclusive scan of the padded count array into the i64 bookmark
// arrays (one segment per list; segments start on tile boundaries and carry
// a trailing zero so bookmark[K] = segment total).  Single pass, decoupled
// look-back restarted at each segment's first tile.
__global__ void __launch_bounds__(kScanThreads) k_lists_scan(const __grid_constant__ ListsParams p,
                                                             const ListsLayout* __restrict__ glay,
                                                             uint64_t* __restrict__ states,
                                                             uint32_t* __restrict__ tile_counter,
                                                             int64_t* __restrict__ seg_totals) {
  __shared__ ListsLayout lay;
  __shared__ int64_t s_tile, s_excl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  load_layout(glay, lay);
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
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
