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

// Segment ids of the count/bookmark arrays: 0 = E2 at max level, l = E4 at l.
struct ListsParams {
  int level;                 // L
  const int64_t* ktot;       // [2*(L+1)]: K_{set,l} at index set*(L+1)+l
  const uint64_t* bmp;       // bitmaps, both sets
  const uint32_t* dir;       // rank directories, same layout
  int64_t bmp_off[2][kMaxLevel + 1];
  const uint64_t* rkeys[kMaxLevel + 1];  // receiver box keys per level < L
  int64_t* bm[kMaxLevel + 1];            // bookmark arrays per segment
  int64_t* ranks_out[kMaxLevel + 1];     // write pass: [0]=E2 list, [l]=E4 ranks
  int16_t* codes_out[kMaxLevel + 1];     // [l]=E4 codes
  // finest-level key window [key_lo, key_hi) owned by this build (the whole
  // grid for a single-GPU build; a Morton range under the multi-GPU
  // partition).  A level-l box is owned when its first finest-level key is.
  uint64_t key_lo, key_hi;
  int dense_rows;  // A/B knob: dense windows written row by row (no line alignment)
};

// Per-level work and segment layout, recomputed per block from the device
// totals (<= 21 levels).
struct ListsLayout {
  int lmin;                     // first level with work
  int64_t work_off[kMaxLevel + 2];  // prefix of receiver-parent counts
  int64_t tile_off[kMaxLevel + 2];  // prefix of count-scan tiles per level
  int64_t r_lo[kMaxLevel + 1];      // owned receiver rows at level l: ranks [r_lo, r_hi)
  int64_t r_hi[kMaxLevel + 1];
  int64_t p_lo[kMaxLevel + 1];      // first receiver parent (rank at level l-1) with an owned row
  int64_t rs_lo[kMaxLevel + 1];     // owned source boxes at level l: ranks [rs_lo, rs_hi)
  int64_t rs_hi[kMaxLevel + 1];
};

constexpr int kCsParents = 64;  // receiver parents per count-scan tile (8 per warp)

__device__ __forceinline__ int lists_lmin(int L) { return L >= 2 ? 2 : L; }

// rank of `key` among the set bits of (set, level l): boxes with smaller keys
__device__ inline int64_t level_rank(const ListsParams& p, int set, int l, uint64_t key) {
  const int L = p.level;
  if (key == 0) return 0;  // (single-GPU windows start at 0: no lookup)
  if (key >= (1ull << (3 * l))) return p.ktot[set * (L + 1) + l];
  const uint64_t* bmp = p.bmp + p.bmp_off[set][l];
  const uint32_t* dir = p.dir + p.bmp_off[set][l];
  const uint64_t w = key >> 6;
  return (int64_t)dir[w] + __popcll(bmp[w] & ((1ull << (key & 63)) - 1ull));
}

__device__ inline void lists_layout(const ListsParams& p, ListsLayout& lay) {
  const int L = p.level;
  lay.lmin = lists_lmin(L);
  int64_t w = 0, t = 0;
  for (int l = 0; l <= kMaxLevel + 1; ++l) lay.work_off[l] = lay.tile_off[l] = 0;
  for (int l = 0; l <= kMaxLevel; ++l)
    lay.r_lo[l] = lay.r_hi[l] = lay.p_lo[l] = lay.rs_lo[l] = lay.rs_hi[l] = 0;
  for (int l = 0; l <= L; ++l) {
    lay.work_off[l] = w;
    lay.tile_off[l] = t;
    const int sh = 3 * (L - l);
    const uint64_t b_lo = (p.key_lo + (1ull << sh) - 1ull) >> sh;  // ceil
    const uint64_t b_hi = (p.key_hi + (1ull << sh) - 1ull) >> sh;
    lay.r_lo[l] = level_rank(p, 1, l, b_lo);
    lay.r_hi[l] = level_rank(p, 1, l, b_hi);
    lay.rs_lo[l] = level_rank(p, 0, l, b_lo);
    lay.rs_hi[l] = level_rank(p, 0, l, b_hi);
    if (l >= lay.lmin) {
      int64_t np;
      if (l == 0) {
        np = p.ktot[(L + 1) + 0];
      } else if (b_hi > b_lo) {
        lay.p_lo[l] = level_rank(p, 1, l - 1, b_lo >> 3);
        np = level_rank(p, 1, l - 1, ((b_hi - 1) >> 3) + 1) - lay.p_lo[l];
      } else {
        np = 0;
      }
      w += np;
      t += (np + kCsParents - 1) / kCsParents;
    }
  }
  lay.work_off[L + 1] = w;
  lay.tile_off[L + 1] = t;
}

__device__ __forceinline__ uint32_t children_mask(const uint64_t* bmp, uint64_t p) {
  return (uint32_t)(__ldg(bmp + (p >> 3)) >> ((int)(p & 7) * 8)) & 0xFFu;
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
  if (threadIdx.x == 0) {
    lists_layout(p, *out);
    // every CSR starts at 0 (levels without receivers get no count-scan tile)
    if (p.level >= 1 && p.bm[0]) p.bm[0][0] = 0;
    for (int l = 2; l <= p.level; ++l)
      if (p.bm[l]) p.bm[l][0] = 0;
  }
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
__device__ __forceinline__ void st_code(unsigned pred, int16_t* c, int code) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.global.s16 [%1], %2;\n\t}" ::
                   "r"(pred), "l"(c), "h"((short)code)
               : "memory");
}
__device__ __forceinline__ void st_rank(unsigned pred, int64_t* r, int64_t rank) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.global.s64 [%1], %2;\n\t}" ::
                   "r"(pred), "l"(r), "l"(rank)
               : "memory");
}

// ---- window order without a sort network.  The Morton order of the 27
// members (x+dx, y+dy, z+dz) of P's window is decided, for a pair of members,
// by the axis with the highest (h * 3 + axis), h = highest differing bit of
// the two coordinates: h(x-1, x) = ctz(x), h(x, x+1) = ctz(x+1) and h(x-1,
// x+1) = the larger of the two.  One of ctz(x), ctz(x+1) is 0, so an axis
// is described by its parity and one level K >= 1, and the whole order by
// the three parities and the ranking of (K_a * 3 + a): 8 x 6 = 48 cases,
// tabulated at compile time from one representative each (members outside
// the grid keep their place and are skipped: no children).
__host__ __device__ constexpr uint64_t cx_morton3(uint64_t x, uint64_t y, uint64_t z) {
  uint64_t k = 0;
  for (int b = 0; b < 21; ++b)
    k |= (((x >> b) & 1ull) << (3 * b)) | (((y >> b) & 1ull) << (3 * b + 1)) |
         (((z >> b) & 1ull) << (3 * b + 2));
  return k;
}
struct WinOrder {
  uint8_t o[48][32];  // [case][sorted position] = window offset (27 = unused)
  constexpr WinOrder() : o() {
    constexpr int ranks[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int cs = 0; cs < 48; ++cs) {
      uint64_t c[3] = {0, 0, 0};
      for (int a = 0; a < 3; ++a) {
        const int K = ranks[cs >> 3][a] + 1;
        c[a] = ((cs >> a) & 1) ? (3ull << K) - 1 : (3ull << K);
      }
      uint64_t key[27] = {};
      int idx[27] = {};
      for (int q = 0; q < 27; ++q) {
        key[q] = cx_morton3(c[0] + q % 3 - 1, c[1] + (q / 3) % 3 - 1, c[2] + q / 9 - 1);
        idx[q] = q;
      }
      for (int i = 0; i < 27; ++i)  // selection sort (compile time)
        for (int j = i + 1; j < 27; ++j)
          if (key[idx[j]] < key[idx[i]]) {
            const int t = idx[i];
            idx[i] = idx[j];
            idx[j] = t;
          }
      for (int i = 0; i < 32; ++i) o[cs][i] = (uint8_t)(i < 27 ? idx[i] : 27);
    }
  }
};
__constant__ WinOrder kWinOrder = WinOrder();

// case of parent P (level l1 >= 0): parities | ranking of (K_a * 3 + a) << 3
__device__ __forceinline__ int window_case(uint64_t P, int l1) {
  const int bits = 3 * l1;
  const uint64_t full = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
  int par = 0, kk[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const uint64_t m = (kDilated << a) & full;
    const uint64_t xa = P & m;
    const int odd = (int)((xa >> a) & 1ull);
    const uint64_t v = odd ? ((((P | ~m) + 1ull) & m)) : xa;  // dilated x+1 or x
    const int K = v ? (__ffsll((long long)v) - 1 - a) / 3 : 64;
    par |= odd << a;
    kk[a] = K * 3 + a;
  }
  const int rx = (kk[0] > kk[1]) + (kk[0] > kk[2]);
  const int ry = (kk[1] > kk[0]) + (kk[1] > kk[2]);
  // (rx, ry) -> index of the ranking in WinOrder's table
  const int pi = rx == 0 ? (ry == 1 ? 0 : 1) : rx == 1 ? (ry == 0 ? 2 : 3) : (ry == 0 ? 4 : 5);
  return par | (pi << 3);
}

// per (window offset o, candidate child c): bits 0-7 near-over-cr (child c of
// o is in the 3x3x3 window of child receiver cr), bits 8+ the E4 code base
// 2*(ox + 7 oy + 49 oz) + (c_x + 7 c_y + 49 c_z) + 171 (minus the receiver's
// own child offset later); o = 27 (unused lanes) is all zero
struct CandTable {
  uint32_t v[28 * 8];
  constexpr CandTable() : v() {
    for (int o = 0; o < 27; ++o) {
      const int off[3] = {o % 3 - 1, (o / 3) % 3 - 1, o / 9 - 1};
      for (int c = 0; c < 8; ++c) {
        uint32_t near = 0;
        for (int cr = 0; cr < 8; ++cr) {
          bool in = true;
          for (int a = 0; a < 3; ++a) {
            const int d = 2 * off[a] + ((c >> a) & 1) - ((cr >> a) & 1);
            in = in && d >= -1 && d <= 1;
          }
          if (in) near |= 1u << cr;
        }
        const int code = 2 * off[0] + 14 * off[1] + 98 * off[2] + (c & 1) + 7 * ((c >> 1) & 1) +
                         49 * ((c >> 2) & 1) + 171;
        v[o * 8 + c] = near | ((uint32_t)code << 8);
      }
    }
  }
};
__constant__ CandTable kCand = CandTable();

// ---- dense windows.  When all 27 window members of a receiver parent are
// in the grid with all 8 children occupied, and all 8 child receivers are
// owned (c2: ~85 % of the finest-level parents), every row's output is a
// fixed sequence: E4 = the 189 candidates outside the child's own window,
// E2 = the 27 inside, in (member slot, child) order, with consecutive source
// ranks per member.  The 8 rows of the parent are consecutive in the CSR
// output, so the parent's whole E4 (E2) output is ONE run of 8 x 189 (8 x 27)
// entries whose candidate sequence and codes depend only on the window case:
// tabulated here (entry = slot * 8 + child), written as line-aligned vector
// stores (dense_run) -- no ballots, no compaction, no partial lines inside a
// run.
constexpr int kDenseE4 = 189, kDenseE2 = 27;
constexpr int kDensePad = 64;  // table padding: a lane pair's out-of-run index reads a valid 0
struct DenseSeq {
  uint8_t e4[48][kDensePad + 8 * kDenseE4 + kDensePad];
  uint8_t e2[48][kDensePad + 8 * kDenseE2 + kDensePad];
  constexpr DenseSeq() : e4(), e2() {
    const WinOrder wo;
    const CandTable ct;
    for (int cs = 0; cs < 48; ++cs) {
      int k4 = kDensePad, k2 = kDensePad;
      for (int cr = 0; cr < 8; ++cr)
        for (int sl = 0; sl < 27; ++sl)
          for (int c = 0; c < 8; ++c) {
            if ((ct.v[wo.o[cs][sl] * 8 + c] >> cr) & 1u)
              e2[cs][k2++] = (uint8_t)(sl * 8 + c);
            else
              e4[cs][k4++] = (uint8_t)(sl * 8 + c);
          }
    }
  }
};
__device__ const DenseSeq kDense = DenseSeq();

__device__ __forceinline__ void st_v2_s64(int64_t* p, int64_t a, int64_t b) {
  asm volatile("st.global.v2.s64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// code offset of child receiver cr: c_x + 7 c_y + 49 c_z
__device__ __forceinline__ int crw_of(int cr) {
  return (cr & 1) + 7 * ((cr >> 1) & 1) + 49 * ((cr >> 2) & 1);
}

// One dense run of n entries: rank = drk[e[k]] (+ its E4 code when CODES:
// the candidate's code base dcd[e] minus the row's child offset).
// Lane pairs (k, k+1) are laid over the output so that every warp store
// covers whole 128-B lines: 64 entries per step = 512 B of ranks in four
// lines (16-B pair stores) and 128 B of codes in one line (4-B pair
// stores); only the first and last lines of the run are partial.
template <bool CODES>
__device__ __forceinline__ void dense_run(int64_t* __restrict__ r, int16_t* __restrict__ c,
                                          const uint8_t* __restrict__ et, int n,
                                          const uint32_t* __restrict__ drk,
                                          const int16_t* __restrict__ dcd, int lane) {
  const uintptr_t ra = (uintptr_t)r >> 3;
  const uintptr_t ca = CODES ? (uintptr_t)c >> 1 : ra;
  const int a = (int)(ca & 63);            // entries before the run in its line
  const bool pair = ((ra ^ ca) & 1) == 0;  // rank pairs 16-B aligned (warp-uniform)
  const int nit = (n + a + 63) >> 6;
  et += kDensePad;  // padded table: indices -64 .. n + 63 are readable
  // E4 row of the pair's first entry, tracked as the pair advances 64
  // entries a step (< 189: at most one row boundary per step)
  int cr = (max(2 * lane - a, 0) * 5549) >> 20;  // k / 189 for k < 1512
  int nb = kDenseE4 * (cr + 1);
  int crw = crw_of(cr), crwn = crw_of(cr + 1);
  constexpr int U = 4;  // steps in flight: table loads, then shared loads, then stores
  for (int it0 = 0; it0 < nit; it0 += U) {
    uint32_t e0[U], e1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k0 = 2 * lane - a + 64 * (it0 + u);
      e0[u] = e1[u] = 0;
      if (it0 + u < nit) {  // (warp-uniform) steps past the run read nothing
        e0[u] = __ldg(et + k0);
        e1[u] = __ldg(et + k0 + 1);
      }
    }
    int64_t v0[U], v1[U];
    int16_t w0[U], w1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v0[u] = (int64_t)drk[e0[u]];
      v1[u] = (int64_t)drk[e1[u]];
      if (CODES) {
        const int k0 = 2 * lane - a + 64 * (it0 + u);
        if (k0 >= nb) {
          ++cr;
          nb += kDenseE4;
          crw = crwn;
          crwn = crw_of(cr + 1);
        }
        w0[u] = (int16_t)(dcd[e0[u]] - crw);
        w1[u] = (int16_t)(dcd[e1[u]] - (k0 + 1 == nb ? crwn : crw));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k0 = 2 * lane - a + 64 * (it0 + u), k1 = k0 + 1;
      const bool ok0 = k0 >= 0 && k0 < n, ok1 = k1 >= 0 && k1 < n;
      if (ok0 && ok1 && pair) {
        st_v2_s64(r + k0, v0[u], v1[u]);
      } else {
        if (ok0) r[k0] = v0[u];
        if (ok1) r[k1] = v1[u];
      }
      if (CODES) {
        if (ok0 && ok1) {
          *reinterpret_cast<uint32_t*>(c + k0) =
              (uint32_t)(uint16_t)w0[u] | ((uint32_t)(uint16_t)w1[u] << 16);
        } else {
          if (ok0) c[k0] = w0[u];
          if (ok1) c[k1] = w1[u];
        }
      }
    }
  }
}

struct ListsSmem {  // per-CTA copies of the tables (lane-divergent lookups)
  uint8_t order[48][32];
  uint32_t cand[28 * 8];
  uint32_t slot[kLWarps][2][32];  // per warp: occupied window members, compacted
  uint32_t dcand[kLWarps][224];    // per warp, dense windows: source rank per candidate ...
  int16_t dcode[kLWarps][224];     // ... and its E4 code base
};
__device__ __forceinline__ void load_tables(ListsSmem& t) {
  for (int i = threadIdx.x; i < 48 * 32 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(&t.order[0][0])[i] =
        reinterpret_cast<const uint32_t*>(&kWinOrder.o[0][0])[i];
  for (int i = threadIdx.x; i < 28 * 8; i += blockDim.x) t.cand[i] = kCand.v[i];
}

// Rows of the owned child receivers (bits of rm, ascending = row order).
// Chunk ch (32 candidates) of row cr: occupied candidates split into E2
// (near cr) and E4 (the rest); both positions come from one ballot of the
// near-and-occupied lanes and the chunk's occupied prefix (shared by the
// rows), and every occupied lane issues ONE rank store (to E2 or E4).
template <bool E4, bool E2>
__device__ __forceinline__ void write_rows(uint32_t rm, int nch, const uint32_t (&meta)[7],
                                           const uint32_t (&rank)[7], int64_t* __restrict__ r4,
                                           int16_t* __restrict__ c4, int64_t* __restrict__ r2) {
  const unsigned lt = lanemask_lt();
  uint32_t oc[7];  // occupied lanes of the chunk: below this lane | total << 8
#pragma unroll
  for (int ch = 0; ch < 7; ++ch) {
    if (ch >= nch) break;  // warp-uniform
    const unsigned ob = ballot_full(meta[ch] & 1u);
    oc[ch] = __popc(ob & lt) | (__popc(ob) << 8);
  }
  uint32_t rbits = rm;
  while (rbits) {
    const int cr = __ffs(rbits) - 1;
    rbits &= rbits - 1;
    const int crw = (cr & 1) + 7 * ((cr >> 1) & 1) + 49 * ((cr >> 2) & 1);
#pragma unroll
    for (int ch = 0; ch < 7; ++ch) {
      if (ch >= nch) break;  // warp-uniform: chunks past the occupied members
      const uint32_t m = meta[ch];
      const uint32_t occ = m & 1u;
      const uint32_t near = (m >> (1 + cr)) & occ;
      const unsigned nb = ballot_full(near);
      const uint32_t a2 = __popc(nb & lt), n2 = __popc(nb);
      const uint32_t a4 = (oc[ch] & 0xFFu) - a2, n4 = (oc[ch] >> 8) - n2;
      if (E2 && E4) {
        int64_t* dst = near ? r2 + a2 : r4 + a4;
        st_rank(occ, dst, (int64_t)rank[ch]);
        st_code(occ & ~near, c4 + a4, (int)(m >> 9) - crw);
      } else if (E4) {
        st_rank_code(occ & ~near, r4 + a4, (int64_t)rank[ch], c4 + a4, (int)(m >> 9) - crw);
      } else {
        st_rank(near, r2 + a2, (int64_t)rank[ch]);
      }
      if (E4) {
        r4 += n4;
        c4 += n4;
      }
      if (E2) r2 += n2;
    }
  }
}

// One receiver parent P (level l-1, rank j among the work parents of level
// l): its rows of E4 (and E2 at l == L).  Lane s holds the s-th window
// member in key order (table, no sort); chunk ch covers members 4ch..4ch+3
// (lane / 8) and their 8 children (lane % 8): occupancy, source rank, the
// near bits over the 8 child receivers and the code base, once per P.
template <bool COMPACT>
__device__ __forceinline__ void write_parent(const ListsParams& p, const ListsLayout& lay,
                                             ListsSmem& t, int L, int l, int64_t j,
                                             int lane) {
  const unsigned FULL = 0xffffffffu;
  const int c = lane & 7;
  const uint64_t P = __ldg(p.rkeys[l - 1] + lay.p_lo[l] + j);
  const int cs = window_case(P, l - 1);
  const int o = t.order[cs][lane];
  const uint64_t qk = window_key(P, l, o);
  uint32_t sm = 0, sfirst = 0;
  if (qk != ~0ull)
    children_of(p.bmp + p.bmp_off[0][l], p.dir + p.bmp_off[0][l], qk, sm, sfirst);
  uint32_t rm, rfirst;
  children_of(p.bmp + p.bmp_off[1][l], p.dir + p.bmp_off[1][l], P, rm, rfirst);
  // owned children (a contiguous run of ranks) and the first one's CSR row
  uint32_t own = 0;
  int64_t r0 = -1;
  if ((int64_t)rfirst >= lay.r_lo[l] && (int64_t)rfirst + __popc(rm) <= lay.r_hi[l]) {
    own = rm;  // the whole run is owned (always, single-GPU)
    r0 = (int64_t)rfirst - lay.r_lo[l];
  } else {
    int64_t r = rfirst;
#pragma unroll
    for (int cb = 0; cb < 8; ++cb)
      if ((rm >> cb) & 1u) {
        if (r >= lay.r_lo[l] && r < lay.r_hi[l]) {
          own |= 1u << cb;
          if (r0 < 0) r0 = r - lay.r_lo[l];
        }
        ++r;
      }
  }
  if (!own) return;
  if (!COMPACT && l >= 2 && own == 0xFFu &&
      __all_sync(FULL, lane >= 27 || sm == 0xFFu)) {  // dense window (see DenseSeq)
    const uint32_t rf = (uint32_t)r0;
    const int64_t g4 = __ldg(p.bm[l] + rf);
    const int64_t g2 = l == L ? __ldg(p.bm[0] + rf) : 0;
    // per candidate e = slot * 8 + child, once for the 8 rows: source rank
    // (consecutive children)
    uint32_t* drk = t.dcand[threadIdx.x >> 5];
    int16_t* dcd = t.dcode[threadIdx.x >> 5];
    __syncwarp();  // the previous parent's reads are done
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      const int e = 32 * k + lane;
      const int sl = e >> 3 < 27 ? e >> 3 : 26;
      drk[e] = __shfl_sync(FULL, sfirst, sl) + (uint32_t)(e & 7);
      dcd[e] = (int16_t)(t.cand[__shfl_sync(FULL, o, sl) * 8 + (e & 7)] >> 8);
    }
    __syncwarp();
    if (p.dense_rows) {
      int64_t* r4 = p.ranks_out[l] + g4;
      int16_t* c4 = p.codes_out[l] + g4;
      int64_t* r2 = l == L ? p.ranks_out[0] + g2 : nullptr;
#pragma unroll 1
      for (int cr = 0; cr < 8; ++cr) {
        const int crw = (cr & 1) + 7 * ((cr >> 1) & 1) + 49 * ((cr >> 2) & 1);
        const uint8_t* q4 = &kDense.e4[cs][kDensePad + cr * kDenseE4];
#pragma unroll
        for (int g = 0; g < 6; ++g) {
          const int tt = 32 * g + lane;
          if (tt < kDenseE4) {
            const uint32_t e = __ldg(q4 + tt);
            r4[tt] = (int64_t)drk[e];
            c4[tt] = (int16_t)(dcd[e] - crw);
          }
        }
        r4 += kDenseE4;
        c4 += kDenseE4;
        if (r2) {
          if (lane < kDenseE2) r2[lane] = (int64_t)drk[__ldg(&kDense.e2[cs][kDensePad + cr * kDenseE2 + lane])];
          r2 += kDenseE2;
        }
      }
      return;
    }
    dense_run<true>(p.ranks_out[l] + g4, p.codes_out[l] + g4, kDense.e4[cs], 8 * kDenseE4, drk,
                    dcd, lane);
    if (l == L)
      dense_run<false>(p.ranks_out[0] + g2, nullptr, kDense.e2[cs], 8 * kDenseE2, drk, dcd,
                       lane);
    return;
  }
  // occupied members compacted in key order (sparse windows -- surfaces,
  // deep levels -- visit ceil(members / 4) chunks instead of 7); per chunk:
  // meta = occ | near-over-cr (8 bits) << 1 | code base << 9
  const unsigned occs = __ballot_sync(FULL, sm != 0u);
  const int nocc = COMPACT ? __popc(occs) : 28;
  // interior with all 27 members occupied: the compacted order is the lane order
  const bool dense = !COMPACT || occs == 0x7FFFFFFu;
  uint32_t* sw = t.slot[threadIdx.x >> 5][0];
  uint32_t* sf = t.slot[threadIdx.x >> 5][1];
  if (!dense) {
    __syncwarp();  // the previous parent's reads are done
    if (sm) {
      const int at = __popc(occs & lanemask_lt());
      sw[at] = sm | ((uint32_t)o << 8);
      sf[at] = sfirst;
    }
    __syncwarp();
  }
  const int nch = (nocc + 3) >> 2;
  const uint32_t slot_word = sm | ((uint32_t)o << 8);
  uint32_t meta[7], rank[7];
#pragma unroll
  for (int ch = 0; ch < 7; ++ch) {
    const int slot = 4 * ch + (lane >> 3);
    const bool in = slot < nocc;  // (!COMPACT: slots >= 27 are the o = 27 lanes)
    uint32_t v, f;
    if (dense) {
      v = __shfl_sync(FULL, slot_word, slot);
      f = __shfl_sync(FULL, sfirst, slot);
    } else {
      v = in ? sw[slot] : (27u << 8);
      f = in ? sf[slot] : 0u;
    }
    const uint32_t smk = v & 0xFFu;
    const uint32_t tv = t.cand[(v >> 8) * 8 + c];
    const bool occ = (smk >> c) & 1u;  // (unused / out-of-grid members: smk = 0)
    meta[ch] = (occ ? 1u : 0u) | ((tv & 0xFFu) << 1) | ((tv >> 8) << 9);
    rank[ch] = f + __popc(smk & ((1u << c) - 1u));
  }
  int64_t* r4 = p.ranks_out[l];
  int16_t* c4 = p.codes_out[l];
  int64_t* r2 = p.ranks_out[0];
  const uint32_t rf = (uint32_t)r0;
  if (l == L) {
    const int64_t w2 = __ldg(p.bm[0] + rf);
    if (l >= 2) {
      const int64_t w4 = __ldg(p.bm[l] + rf);
      write_rows<true, true>(own, nch, meta, rank, r4 + w4, c4 + w4, r2 + w2);
    } else {
      write_rows<false, true>(own, nch, meta, rank, nullptr, nullptr, r2 + w2);
    }
  } else {
    const int64_t w4 = __ldg(p.bm[l] + rf);
    write_rows<true, false>(own, nch, meta, rank, r4 + w4, c4 + w4, nullptr);
  }
}

// COMPACT: occupied window members compacted first (sparse levels; the host
// picks it from the count pass's entries per row), else the dense layout
#ifndef FMMB_LW_MINB
#define FMMB_LW_MINB 4
#endif
template <bool COMPACT>
__global__ void __launch_bounds__(kLThreads, FMMB_LW_MINB)
    k_lists_write(const __grid_constant__ ListsParams p, const ListsLayout* __restrict__ glay) {
  __shared__ ListsLayout lay;
  __shared__ ListsSmem tab;
  load_layout(glay, lay);
  load_tables(tab);
  __syncthreads();
  const int L = p.level;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwork = lay.work_off[L + 1];
  const int64_t gstride = (int64_t)gridDim.x * kLWarps;
  for (int64_t gw = (int64_t)blockIdx.x * kLWarps + warp; gw < nwork; gw += gstride) {
    int l = lay.lmin;
    while (lay.work_off[l + 1] <= gw) ++l;
    const int64_t j = gw - lay.work_off[l];
    if (l == 0) {
      if (lane == 0 && p.ktot[0]) p.ranks_out[0][p.bm[0][0]] = 0;
      continue;
    }
    write_parent<COMPACT>(p, lay, tab, L, l, j, lane);
  }
}

// Count + CSR scan in one pass.  A tile is kCsParents consecutive receiver
// parents P of one level (8 per warp); for each child receiver r of P it
// counts |E4_l(r)| (and |E2(r)| at l == L) -- lane = window slot, the
// near-children counts of all 8 children from one SWAR byte-popcount and two
// warp reductions -- then the tile's rows (children in P order = ascending
// receiver keys) are scanned in shared memory and offset by a decoupled
// look-back over the level's tiles (tickets keep tiles in order).  Writes
// the bookmark arrays and the per-level totals.
template <bool PERSISTENT>
__global__ void __launch_bounds__(kLThreads)
    k_lists_cscan(const __grid_constant__ ListsParams p, const ListsLayout* __restrict__ glay,
                  uint64_t* __restrict__ st4, uint64_t* __restrict__ st2,
                  uint32_t* __restrict__ ticket, int64_t* __restrict__ seg_totals) {
  __shared__ ListsLayout lay;
  __shared__ uint32_t s_rm[kCsParents], s_rf[kCsParents];
  __shared__ uint16_t s_c4[kCsParents * 8], s_c2[kCsParents * 8];
  __shared__ uint32_t s_w4[kLWarps], s_w2[kLWarps];
  __shared__ int64_t s_tile, s_b4, s_b2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  load_layout(glay, lay);
  const int L = p.level;
  // one tile per CTA, or (PERSISTENT: the per-level bounds the grid is sized
  // from before the totals are known are loose -- c3: 300 K bound tiles, 5 K
  // real ones) tiles taken by ticket until none is left
  for (;;) {
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  if (L == 0) {  // the root receiver sees the root source
    if (tile == 0 && tid == 0) {
      const int64_t kr = p.ktot[1], e2 = kr ? p.ktot[0] : 0;
      p.bm[0][0] = 0;
      if (kr) p.bm[0][1] = e2;
      seg_totals[0] = e2;
    }
    return;
  }
  if (tile >= lay.tile_off[L + 1]) return;
  int l = lay.lmin;
  while (lay.tile_off[l + 1] <= tile) ++l;
  const int64_t first_tile = lay.tile_off[l];
  const int64_t np = lay.work_off[l + 1] - lay.work_off[l];
  const int64_t j0 = (tile - first_tile) * kCsParents;
  const unsigned FULL = 0xffffffffu;
  const uint64_t nearw = lane < 27 ? kNear.w[lane] : 0ull;
  constexpr int kPW = kCsParents / kLWarps;
  for (int k = 0; k < kPW; ++k) {
    const int pi = warp * kPW + k;
    const int64_t j = j0 + pi;
    uint32_t rm = 0, rfirst = 0, sm = 0;
    if (j < np) {
      const uint64_t P = __ldg(p.rkeys[l - 1] + lay.p_lo[l] + j);
      const uint64_t qk = window_key(P, l, lane);
      if (qk != ~0ull) sm = children_mask(p.bmp + p.bmp_off[0][l], qk);
      children_of(p.bmp + p.bmp_off[1][l], p.dir + p.bmp_off[1][l], P, rm, rfirst);
    }
    const uint64_t e2b = popc_bytes(((uint64_t)sm * 0x0101010101010101ull) & nearw);
    const uint32_t lo = __reduce_add_sync(FULL, (uint32_t)e2b);
    const uint32_t hi = __reduce_add_sync(FULL, (uint32_t)(e2b >> 32));
    const uint32_t all = __reduce_add_sync(FULL, (uint32_t)__popc(sm));
    if (lane < 8) {
      const uint32_t e2 = ((lane < 4 ? lo >> (8 * lane) : hi >> (8 * (lane - 4)))) & 0xFFu;
      const int64_t row = (int64_t)rfirst + __popc(rm & ((1u << lane) - 1u));
      const bool has = ((rm >> lane) & 1u) && row >= lay.r_lo[l] && row < lay.r_hi[l];
      s_c4[pi * 8 + lane] = (uint16_t)(has && l >= 2 ? all - e2 : 0u);
      s_c2[pi * 8 + lane] = (uint16_t)(has ? e2 : 0u);
    }
    if (lane == 0) {
      s_rm[pi] = rm;
      s_rf[pi] = rfirst;
    }
  }
  __syncthreads();
  // exclusive scan over the tile's 64 x 8 child slots (empty slots count 0)
  uint32_t a4 = s_c4[2 * tid], b4 = s_c4[2 * tid + 1];
  uint32_t a2 = s_c2[2 * tid], b2 = s_c2[2 * tid + 1];
  uint32_t t4, t2;
  uint32_t x4 = warp_excl_scan(a4 + b4, t4);
  uint32_t x2 = warp_excl_scan(a2 + b2, t2);
  if (lane == 0) {
    s_w4[warp] = t4;
    s_w2[warp] = t2;
  }
  __syncthreads();
  uint32_t tot4 = 0, tot2 = 0;
#pragma unroll
  for (int i = 0; i < kLWarps; ++i) {
    x4 += i < warp ? s_w4[i] : 0u;
    x2 += i < warp ? s_w2[i] : 0u;
    tot4 += s_w4[i];
    tot2 += s_w2[i];
  }
  const bool last = tile == lay.tile_off[l + 1] - 1;
  // warp 0 looks back over the E4 states, warp 1 over the E2 states
  if (warp < 2) {
    const bool on = warp == 0 ? l >= 2 : l == L;
    uint64_t* sts = warp == 0 ? st4 : st2;
    const uint64_t tot = warp == 0 ? tot4 : tot2;
    uint64_t e = 0;
    if (on) {
      if (tile == first_tile) {
        if (lane == 0) st_state(sts + tile, kStInclusive | tot);
      } else {
        if (lane == 0) st_state(sts + tile, kStAggregate | tot);
        e = lookback_warp(sts, tile, first_tile, 1);
        if (lane == 0) st_state(sts + tile, kStInclusive | (e + tot));
      }
    }
    if (lane == 0) (warp == 0 ? s_b4 : s_b2) = (int64_t)e;
  }
  __syncthreads();
  const int64_t base4 = s_b4, base2 = s_b2;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int slot = 2 * tid + e;
    const int pi = slot >> 3, c = slot & 7;
    const uint32_t rm = s_rm[pi];
    const int64_t row = (int64_t)s_rf[pi] + __popc(rm & ((1u << c) - 1u)) - lay.r_lo[l];
    if (((rm >> c) & 1u) && row >= 0 && row < lay.r_hi[l] - lay.r_lo[l]) {
      if (l >= 2) p.bm[l][row] = base4 + x4;
      if (l == L) p.bm[0][row] = base2 + x2;
    }
    x4 += e == 0 ? a4 : b4;
    x2 += e == 0 ? a2 : b2;
  }
  if (last && tid == 0) {  // trailing bookmark = segment total
    const int64_t kr = lay.r_hi[l] - lay.r_lo[l];
    if (l >= 2) {
      p.bm[l][kr] = base4 + tot4;
      seg_totals[l] = base4 + tot4;
    }
    if (l == L) {
      p.bm[0][kr] = base2 + tot2;
      seg_totals[0] = base2 + tot2;
    }
  }
  if (!PERSISTENT) return;
  __syncthreads();  // shared state reused by the next tile
  }
}

}  // namespace fmmb
