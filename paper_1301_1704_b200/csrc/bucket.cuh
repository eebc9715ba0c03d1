// Sort side of the build, payload-carrying bucket sort (the fast path).
//
// Reference semantics reproduced: pseudosort.histogram_and_sort_index +
// reorder + build_bookmarks (pseudosort.py:41-135), i.e. the permutation is
// np.argsort(keys, kind="stable") (tests/test_pseudosort.py:94-104) with the
// compiled backend's encode (_ckernels.pyx:85-104).  A bucket is a contiguous
// range of Morton keys (the top `bb` key bits of one set), so the sorted
// buckets concatenated are the global order and no box straddles two buckets.
//
//   H  k_bkt_hist    : read xyz once; per-CTA histogram of the bucket ids in
//                      shared memory, one row per CTA.
//   S  k_bkt_scan    : column sums, exclusive scan -> bucket starts; the
//                      starts seed one global cursor per bucket.
//   S  k_bkt_scatter : read xyz(+q) again, streamed through a shared-memory
//                      ring by TMA bulk copies; every point claims a slot at
//                      its bucket's cursor (one atomic per point) and is
//                      written there as a 32-byte record {x, y, z, q | recv
//                      index} (+ its source index).  Cursors advance in time,
//                      so every bucket fills front to back and L2 merges the
//                      partial lines; the order inside a bucket is arbitrary.
//   L  k_bkt_local   : one CTA per bucket: TMA bulk copy of the bucket's
//                      records into shared memory, then a sort by (low key
//                      bits, combined input index) -- the index makes the
//                      order the stable one whatever the arrival order was --
//                      and the reference layout (points, charges,
//                      permutation, boxes); box heads give the bookmarks,
//                      non-empty keys and level-L occupancy bits.
//
// DRAM bytes per point (src / recv): H 24/24, S 32+36 / 24+32, L 36+48 / 32+40.
//
// The fast path needs every bucket to fit the local sort's shared memory
// (kLcCap points); buckets hold <= 1024 points on average by construction.
// Skewed inputs (dense clusters) overflow it: the local kernel then raises
// `fail` and the host reruns the sort phase on the general Onesweep path
// (sort.cuh + finalize.cuh).
#pragma once
#include "common.cuh"

namespace fmmb {

constexpr int kBucketBitsMax = 14;  // <= 2^14 buckets per set
constexpr int kBucketAvg = 1024;    // bb chosen so the mean bucket is <= this
constexpr int kHThreads = 512;      // H pass
constexpr int kHItems = 8;          // rows per lane per step (memory-level parallelism)
constexpr int kHChunk = 32 * kHItems;

constexpr int kScanBuckets = 1024;  // buckets per CTA of the scan
constexpr int kCursorStride = 32;   // u32 words per bucket cursor: one 128-B line each, so
                                    // the scatter's cursor atomics never share an L2 line

struct BucketGeo {
  int sbits;      // 3L
  int bb;         // bucket bits per set
  int shift;      // 3L - bb: low key bits sorted inside a bucket
  int nb;         // 2 << bb buckets
  int64_t n, m;   // sources, receivers
  int cbits;      // bits of a combined input index (n + m <= 2^cbits)
  int hgrid;      // CTAs (histogram rows) of the H pass
  int qrec;       // source records carry the charge ({x, y, z, q}) and the source
                  // index goes to the idx side array at the same slot; else the
                  // record carries the index and k_gather_q sorts the charges
  int eb;         // qrec: bits per coordinate exponent of the index embedding
                  // (0: none; see rec_embed)
};

// Source records {x, y, z, q} have no room for the input index, but a
// coordinate v in [2^-(2^eb), 1) is fully described by its 52-bit mantissa
// and e = -1 - floor(log2 v) < 2^eb: the record then stores the mantissas
// and moves the three sign+exponent fields (36 bits) into a payload of
// cbits index bits + 3 eb exponent bits, flagged by x's sign bit and bit 52
// (raw coordinates with that pattern are negative: a DomainError input).
// Points with any coordinate outside that range (rare: 3 / 256 of uniform
// points at eb = 3) keep raw coordinates and the idx side store.
__device__ __forceinline__ bool rec_embed(double& x, double& y, double& z, uint32_t ci,
                                          const BucketGeo& g) {
  if (!g.eb) return false;
  const uint64_t lo = (uint64_t)(1023 - (1 << g.eb)) << 52;  // bits of 2^-(2^eb)
  const uint64_t span = (1023ull << 52) - lo;                 // up to 1.0 (excl.)
  const uint64_t bx = (uint64_t)__double_as_longlong(x), by = (uint64_t)__double_as_longlong(y),
                 bz = (uint64_t)__double_as_longlong(z);
  if (bx - lo >= span || by - lo >= span || bz - lo >= span) return false;
  const uint64_t m52 = (1ull << 52) - 1ull;
  const uint64_t ex = 1022 - (bx >> 52), ey = 1022 - (by >> 52), ez = 1022 - (bz >> 52);
  const uint64_t pay = (uint64_t)ci | (ex << g.cbits) | (ey << (g.cbits + g.eb)) |
                       (ez << (g.cbits + 2 * g.eb));  // < 2^34
  x = __longlong_as_double((long long)((1ull << 63) | ((((pay & 0x3FFull) << 1) | 1ull) << 52) |
                                       (bx & m52)));
  y = __longlong_as_double((long long)((((pay >> 10) & 0xFFFull) << 52) | (by & m52)));
  z = __longlong_as_double((long long)((((pay >> 22) & 0xFFFull) << 52) | (bz & m52)));
  return true;
}

// inverse of rec_embed on a source record: restores x, y, z, returns the
// index; false (and nothing touched) for a raw record
__device__ __forceinline__ bool rec_extract(double* r, uint32_t& ci, const BucketGeo& g) {
  const uint64_t bx = (uint64_t)__double_as_longlong(r[0]);
  if (!g.eb || !(bx >> 63) || !((bx >> 52) & 1ull)) return false;
  const uint64_t by = (uint64_t)__double_as_longlong(r[1]), bz = (uint64_t)__double_as_longlong(r[2]);
  const uint64_t m52 = (1ull << 52) - 1ull;
  const uint64_t pay = ((bx >> 53) & 0x3FFull) | (((by >> 52) & 0xFFFull) << 10) |
                       (((bz >> 52) & 0xFFFull) << 22);
  const uint64_t em = (1ull << g.eb) - 1ull;
  const uint64_t ex = (pay >> g.cbits) & em, ey = (pay >> (g.cbits + g.eb)) & em,
                 ez = (pay >> (g.cbits + 2 * g.eb)) & em;
  ci = (uint32_t)(pay & ((1ull << g.cbits) - 1ull));
  r[0] = __longlong_as_double((long long)(((1022 - ex) << 52) | (bx & m52)));
  r[1] = __longlong_as_double((long long)(((1022 - ey) << 52) | (by & m52)));
  r[2] = __longlong_as_double((long long)(((1022 - ez) << 52) | (bz & m52)));
  return true;
}

__host__ inline int ceil_log2(int64_t v) {
  int b = 0;
  while (b < 62 && (1ll << b) < v) ++b;
  return b;
}

__host__ inline BucketGeo bucket_geo(int level, int64_t n, int64_t m, int num_sms) {
  BucketGeo g{};
  g.sbits = 3 * level;
  const int64_t nmax = n > m ? n : m;
  int bb = ceil_log2((nmax + kBucketAvg - 1) / kBucketAvg);
  if (bb > kBucketBitsMax) bb = kBucketBitsMax;
  if (bb > g.sbits) bb = g.sbits;
  g.bb = bb;
  g.shift = g.sbits - bb;
  g.nb = 2 << bb;
  g.n = n;
  g.m = m;
  const int64_t tot = n + m;
  g.cbits = ceil_log2(tot > 1 ? tot : 2);
  const int64_t hchunks = (tot + (int64_t)kHThreads * kHItems - 1) / ((int64_t)kHThreads * kHItems);
  g.hgrid = (int)(hchunks < num_sms ? (hchunks < 1 ? 1 : hchunks) : num_sms);
  return g;
}

// rows of the combined [src | recv] input: point i < n is src[i], else recv[i-n]
__device__ __forceinline__ const double* row_ptr(const double* src, const double* recv,
                                                 int64_t n, int64_t i) {
  return i < n ? src + 3 * i : recv + 3 * (i - n);
}

__device__ __forceinline__ uint32_t bucket_of(uint64_t key, int is_recv, const BucketGeo& g) {
  return ((uint32_t)is_recv << g.bb) | (uint32_t)(key >> g.shift);
}

// ---------------------------------------------------------------- H pass --
// With `fine` non-null (wide geometries, where every non-empty coarse bucket
// is refined) the same read also counts every point's refinement sub-bin
// (global atomics into fine[bucket][sub]), so k_bkt_fine's second read of the
// inputs is skipped.  With bmp_src / bmp_recv non-null the pass also sets the
// level-L occupancy bits, so the directory and the lists can start while the
// scatter and the local pass still run (build.cu, early occupancy).
template <bool NARROW>
__global__ void __launch_bounds__(kHThreads)
    k_bkt_hist(const double* __restrict__ src, const double* __restrict__ recv,
               const BucketGeo g, int level, uint32_t* __restrict__ mat,
               uint32_t* __restrict__ err, uint32_t* __restrict__ fine,
               unsigned long long* __restrict__ bmp_src,
               unsigned long long* __restrict__ bmp_recv) {
  extern __shared__ uint32_t s_hist[];  // [nb]
  const int lane = threadIdx.x & 31;
  for (int b = threadIdx.x; b < g.nb; b += kHThreads) s_hist[b] = 0;
  __syncthreads();
  const int64_t tot = g.n + g.m;
  const uint64_t lim = 1ull << g.sbits;
  const double grid = (double)(1ll << level);
  bool bad = false;
  const int64_t wstride = (int64_t)g.hgrid * (kHThreads / 32);
  for (int64_t c = (int64_t)blockIdx.x * (kHThreads / 32) + (threadIdx.x >> 5);
       c * kHChunk < tot; c += wstride) {
    const int64_t base = c * kHChunk;
    double x[kHItems], y[kHItems], z[kHItems];
#pragma unroll
    for (int k = 0; k < kHItems; ++k) {
      const int64_t i = base + k * 32 + lane;
      if (i < tot) {
        const double* p = row_ptr(src, recv, g.n, i);
        x[k] = __ldg(p);
        y[k] = __ldg(p + 1);
        z[k] = __ldg(p + 2);
      }
    }
#pragma unroll
    for (int k = 0; k < kHItems; ++k) {
      const int64_t i = base + k * 32 + lane;
      if (i < tot) {
        const uint64_t key = encode_any<NARROW>(x[k], y[k], z[k], level, grid);
        bad |= key >= lim;
        const uint32_t b = bucket_of(key & (lim - 1), i >= g.n, g);
        atomicAdd(&s_hist[b], 1u);
        if (bmp_src) {  // level-L occupancy bit (fire-and-forget reduction)
          const uint64_t k = key & (lim - 1);
          unsigned long long* w = (i >= g.n ? bmp_recv : bmp_src) + (k >> 6);
          asm volatile("red.global.or.b64 [%0], %1;" ::"l"(w), "l"(1ull << (k & 63)) : "memory");
        }
        if (fine) {
          const int R = g.shift < 8 ? g.shift : 8;  // = ref_bits(g)
          const uint32_t sub = (uint32_t)(((key & (lim - 1)) >> (g.shift - R)) & ((1u << R) - 1u));
          atomicAdd(fine + (size_t)b * 256 + sub, 1u);  // 256 = kRefBins
        }
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 1u);
  __syncthreads();
  uint32_t* row = mat + (size_t)blockIdx.x * g.nb;
  for (int b = threadIdx.x; b < g.nb; b += kHThreads) row[b] = s_hist[b];
}

// ------------------------------------------------------------- scan pass --
// CTA = kScanBuckets buckets in order (ticket + decoupled look-back).
// bstart[b] = first sorted position of bucket b (bstart[nb] = n + m),
// *maxb = largest bucket.
__global__ void __launch_bounds__(256)
    k_bkt_scan(const uint32_t* __restrict__ mat, const BucketGeo g, uint32_t* __restrict__ bstart,
               uint64_t* __restrict__ states,
               uint32_t* __restrict__ ticket, uint32_t* __restrict__ maxb) {
  constexpr int kPer = kScanBuckets / 256;
  __shared__ uint32_t s_w[8];
  __shared__ int64_t s_tile, s_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int b0 = (int)tile * kScanBuckets + threadIdx.x * kPer;
  uint32_t c[kPer];
  uint32_t tsum = 0, tmax = 0;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    c[e] = 0;
    const int b = b0 + e;
    if (b < g.nb)
      for (int r = 0; r < g.hgrid; ++r) c[e] += __ldg(mat + (size_t)r * g.nb + b);
    tsum += c[e];
    tmax = c[e] > tmax ? c[e] : tmax;
  }
  tmax = __reduce_max_sync(0xffffffffu, tmax);
  if (lane == 0 && tmax) atomicMax(maxb, tmax);
  uint32_t wt;
  uint32_t x = warp_excl_scan(tsum, wt);
  if (lane == 0) s_w[warp] = wt;
  __syncthreads();
  uint32_t all = 0;
  for (int i = 0; i < 8; ++i) {
    x += i < warp ? s_w[i] : 0u;
    all += s_w[i];
  }
  if (threadIdx.x == 0) {
    uint64_t* st = states + tile;
    uint64_t excl = 0;
    if (tile == 0) {
      st_state(st, kStInclusive | all);
    } else {
      st_state(st, kStAggregate | all);
      excl = lookback(states, tile, 0, 1);
      st_state(st, kStInclusive | (excl + all));
    }
    s_base = (int64_t)excl;
    if ((int64_t)(tile + 1) * kScanBuckets >= g.nb) bstart[g.nb] = (uint32_t)(excl + all);
  }
  __syncthreads();
  uint32_t run = (uint32_t)s_base + x;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    const int b = b0 + e;
    if (b < g.nb) bstart[b] = run;
    run += c[e];
  }
}

// ------------------------------------------------------- refinement ----
// Skewed inputs (a coarse bucket holds more points than the local sort's
// shared memory) are handled by splitting every such bucket along the next
// kRefBits key bits: a fine histogram of the big buckets' points, then a
// greedy grouping of consecutive sub-bins into FINAL buckets of <= kLcCap
// points.  A final bucket is a contiguous key range [lo, lo + span); uniform
// inputs keep final == coarse buckets (nothing is refined).
constexpr int kRefBits = 8;
constexpr int kLcSmallBits_ = 11;  // = kLcSmallBits (box-count path span)
constexpr int kRefBins = 1 << kRefBits;

struct BDesc {          // final bucket: level-L key range and set
  uint64_t lo;
  uint64_t span_set;    // span | set << 63
};

__host__ inline int64_t final_buckets_cap(const BucketGeo& g, int64_t cap) {
  // greedy groups: two neighbours hold > cap points or a neighbour is a full
  // run of sub-bins, so groups <= 2 * points / cap + 2 * runs + 1 per bucket
  const int R = g.shift < kRefBits ? g.shift : kRefBits;
  const int sh_sub = g.shift - R;
  const int64_t runs = sh_sub >= 11 ? (1 << R) : ((1 << R) >> (11 - sh_sub));
  return (int64_t)g.nb * (1 + 2 * std::max<int64_t>(runs, 1)) + 3 * ((g.n + g.m) / cap + 1);
}

__device__ __forceinline__ int ref_bits(const BucketGeo& g) {
  return g.shift < kRefBits ? g.shift : kRefBits;
}

// a coarse bucket is refined when it holds more points than the local sort's
// shared memory, or when its key span is too wide for the box-count path
// (then final buckets are also capped at 2^kLcSmallBits keys)
__device__ __forceinline__ bool wide_buckets(const BucketGeo& g) {
  return g.shift > kLcSmallBits_;
}
__device__ __forceinline__ bool needs_refine(const BucketGeo& g, uint32_t count, uint32_t cap) {
  return count > cap || (wide_buckets(g) && count > 0);
}

// fine histogram of the points of over-full coarse buckets (a no-op grid when
// every bucket fits)
template <bool NARROW>
__global__ void __launch_bounds__(256)
    k_bkt_fine(const double* __restrict__ src, const double* __restrict__ recv,
               const BucketGeo g, int level, const uint32_t* __restrict__ bstart,
               const uint32_t* __restrict__ maxb, uint32_t cap, uint32_t* __restrict__ fine) {
  // nothing to refine, or wide geometry (the H pass already counted the sub-bins)
  if ((__ldg(maxb) <= cap && !wide_buckets(g)) || wide_buckets(g)) return;
  const int64_t tot = g.n + g.m;
  const uint64_t kmask = (1ull << g.sbits) - 1ull;
  const double grid = (double)(1ll << level);
  const int R = ref_bits(g);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* p = row_ptr(src, recv, g.n, i);
    const uint64_t key = encode_any<NARROW>(__ldg(p), __ldg(p + 1), __ldg(p + 2), level, grid) & kmask;
    const uint32_t b = bucket_of(key, i >= g.n, g);
    if (needs_refine(g, __ldg(bstart + b + 1) - __ldg(bstart + b), cap)) {
      const uint32_t sub = (uint32_t)((key >> (g.shift - R)) & ((1u << R) - 1u));
      atomicAdd(fine + (size_t)b * kRefBins + sub, 1u);
    }
  }
}

// Final buckets: thread per coarse bucket (CTA = 256 buckets, tickets +
// decoupled look-back for the final-bucket numbering).  Writes fbase[b],
// the sub-bin -> group table of refined buckets, every final bucket's start,
// descriptor and scatter cursor, and nfinal.
struct PlanOut {
  uint32_t* fbase;   // [nb]
  uint8_t* gtab;     // [nb * kRefBins]
  uint32_t* bstart_f;  // [nfinal + 1]
  BDesc* desc;       // [nfinal]
  uint32_t* cursor;  // [nfinal * kCursorStride]
  uint32_t* nfinal;  // [1]
  uint32_t* fail;    // [1]
  uint64_t* states;  // [nb / 256 + 1]
  uint32_t* ticket;  // [1]
};

__global__ void __launch_bounds__(256)
    k_bkt_plan(const BucketGeo g, const uint32_t* __restrict__ bstart,
               const uint32_t* __restrict__ maxb, uint32_t cap,
               const uint32_t* __restrict__ fine, const PlanOut o) {
  __shared__ uint32_t s_w[8];
  __shared__ int64_t s_tile, s_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(o.ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int b = (int)tile * 256 + tid;
  const bool refined = __ldg(maxb) > cap || wide_buckets(g);
  const int R = ref_bits(g);
  const int nsub = 1 << R;
  // sub-bins per final bucket: its key span stays within the count path
  const int sh_sub = g.shift - R;
  const int max_run = sh_sub >= kLcSmallBits_ ? 1 : (1 << (kLcSmallBits_ - sh_sub));
  uint32_t c = 0, ns = 0;
  if (b < g.nb) {
    c = bstart[b + 1] - bstart[b];
    ns = 1;
    if (refined && needs_refine(g, c, cap)) {  // greedy groups of consecutive sub-bins
      // (sub-bin counts streamed 4 at a time, group ids stored 4 per word)
      const uint32_t* f = fine + (size_t)b * kRefBins;
      uint8_t* gt = o.gtab + (size_t)b * kRefBins;
      uint32_t acc = 0, grp = 0;
      int run = 0;
      bool over = false;
      for (int q4 = 0; q4 < (nsub + 3) / 4; ++q4) {
        const uint4 v4 = nsub >= 4 ? __ldg(reinterpret_cast<const uint4*>(f) + q4)
                                   : make_uint4(f[0], nsub > 1 ? f[1] : 0u, 0u, 0u);
        const uint32_t vv[4] = {v4.x, v4.y, v4.z, v4.w};
        uint32_t packed = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (4 * q4 + e >= nsub) break;
          const uint32_t v = vv[e];
          over |= v > cap;
          if ((acc + v > cap && acc > 0) || run == max_run) {
            ++grp;
            acc = 0;
            run = 0;
          }
          acc += v;
          ++run;
          packed |= (grp & 0xFFu) << (8 * e);
        }
        if (nsub >= 4) reinterpret_cast<uint32_t*>(gt)[q4] = packed;
        else for (int e = 0; e < nsub; ++e) gt[e] = (uint8_t)(packed >> (8 * e));
      }
      if (over) atomicOr(o.fail, 1u);
      ns = grp + 1;
    }
  }
  uint32_t wt;
  uint32_t x = warp_excl_scan(ns, wt);
  if (lane == 0) s_w[warp] = wt;
  __syncthreads();
  uint32_t all = 0;
  for (int i = 0; i < 8; ++i) {
    x += i < warp ? s_w[i] : 0u;
    all += s_w[i];
  }
  if (tid == 0) {
    uint64_t* st = o.states + tile;
    uint64_t excl = 0;
    if (tile == 0) {
      st_state(st, kStInclusive | all);
    } else {
      st_state(st, kStAggregate | all);
      excl = lookback(o.states, tile, 0, 1);
      st_state(st, kStInclusive | (excl + all));
    }
    s_base = (int64_t)excl;
    if ((int64_t)(tile + 1) * 256 >= g.nb) {
      *o.nfinal = (uint32_t)(excl + all);
      o.bstart_f[excl + all] = (uint32_t)(g.n + g.m);
    }
  }
  __syncthreads();
  if (b >= g.nb) return;
  const uint32_t fb = (uint32_t)s_base + x;
  o.fbase[b] = fb;
  const uint64_t set = (uint64_t)(b >> g.bb);
  const uint64_t lo = (uint64_t)(b & ((1 << g.bb) - 1)) << g.shift;
  if (ns == 1) {
    o.bstart_f[fb] = bstart[b];
    o.desc[fb] = BDesc{lo, (1ull << g.shift) | (set << 63)};
    o.cursor[(size_t)fb * kCursorStride] = bstart[b];
    return;
  }
  // the same greedy walk again, emitting each group's start, key range and
  // cursor (no read-back of the group table)
  const uint32_t* f = fine + (size_t)b * kRefBins;
  const int sh = g.shift - R;
  uint32_t start = bstart[b];
  uint32_t acc = 0, grp = 0;
  int run = 0, first = 0;
  auto emit = [&](int end) {
    const uint32_t fid = fb + grp;
    o.bstart_f[fid] = start;
    o.desc[fid] = BDesc{lo + ((uint64_t)first << sh), ((uint64_t)(end - first) << sh) | (set << 63)};
    o.cursor[(size_t)fid * kCursorStride] = start;
    start += acc;
  };
  for (int q4 = 0; q4 < (nsub + 3) / 4; ++q4) {
    const uint4 v4 = nsub >= 4 ? __ldg(reinterpret_cast<const uint4*>(f) + q4)
                               : make_uint4(f[0], nsub > 1 ? f[1] : 0u, 0u, 0u);
    const uint32_t vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int sb = 4 * q4 + e;
      if (sb >= nsub) break;
      const uint32_t v = vv[e];
      if ((acc + v > cap && acc > 0) || run == max_run) {
        emit(sb);
        ++grp;
        acc = 0;
        run = 0;
        first = sb;
      }
      acc += v;
      ++run;
    }
  }
  emit(nsub);
}

// ------------------------------------------------ speculative regions ----
// Uniform inputs skip the histogram pass: every coarse bucket gets a region of
// kLcCap record slots (the local sort's capacity), the scatter claims slots
// from region cursors, and the exact output starts come from the final
// cursors afterwards.  A region overflow (a skewed input) raises spec_fail
// and the host reruns the sort phase with the histogram pass.  Regions are
// kSpecStride (odd) records apart, so the 2^15 region fronts do not all fall
// on the same DRAM / L2 address bits.
constexpr int kSpecStride = 1281;
__global__ void __launch_bounds__(256)
    k_spec_init(const BucketGeo g, uint32_t cap, uint32_t* __restrict__ cursor,
                uint32_t* __restrict__ rbase, BDesc* __restrict__ desc,
                uint32_t* __restrict__ nfinal) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) *nfinal = (uint32_t)g.nb;
  if (b >= g.nb) return;
  cursor[(size_t)b * kCursorStride] = (uint32_t)b * cap;
  rbase[b] = (uint32_t)b * cap;
  const uint64_t set = (uint64_t)(b >> g.bb);
  desc[b] = BDesc{(uint64_t)(b & ((1 << g.bb) - 1)) << g.shift, (1ull << g.shift) | (set << 63)};
}

// region fill counts, in the layout k_bkt_scan sums (one histogram row)
__global__ void __launch_bounds__(256)
    k_spec_counts(const BucketGeo g, uint32_t cap, const uint32_t* __restrict__ cursor,
                  uint32_t* __restrict__ counts) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nb) return;
  const uint32_t c = cursor[(size_t)b * kCursorStride] - (uint32_t)b * cap;
  counts[b] = c < cap ? c : cap;
}

// ---------------------------------------------------------- scatter pass --
__device__ __forceinline__ void st_v4f64(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d)
               : "memory");
}

// mbarrier / bulk-copy helpers (TMA 1-D bulk copies, sm_90+ / sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// S pass.  One persistent CTA per SM streams a contiguous input range
// through a kSStages-deep shared-memory ring of kSRows-row stages filled by
// TMA bulk copies (thread 0 produces).  Thread t owns row t of every stage:
// it claims the row's bucket slot with one atomic, and stores the record
// kSDepth stages later straight from the ring, so the atomic round trip
// overlaps the following stages and the payload never sits in registers;
// the stage is released (`empty` mbarrier) after that store.  Stages that
// straddle the src/recv boundary or are not 16-byte aligned are filled by
// their consumers with plain loads instead.
constexpr int kSThreads = 1024;
constexpr int kSRows = kSThreads;   // one row per thread per stage
#ifndef FMMB_SLEAD  // scatter pipeline shape (overridable for measurement builds)
#define FMMB_SLEAD 3
#define FMMB_SDEPTH 2
#define FMMB_SSTAGES 6
#endif
constexpr int kSStages = FMMB_SSTAGES;
constexpr int kSLead = FMMB_SLEAD;    // stages in flight ahead of the claim
constexpr int kSDepth = FMMB_SDEPTH;  // stages between claim and store
static_assert(kSLead + kSDepth + 1 <= kSStages, "ring too small");
constexpr int kSStageBytes = kSRows * 32;  // xyz (24 B) + q (8 B) per row

__host__ __device__ constexpr size_t scatter_smem_bytes() {
  return (size_t)kSStages * kSStageBytes + 2 * kSStages * 8;
}

__host__ inline int64_t scatter_rows_per_cta(int64_t tot, int grid) {
  int64_t r = (tot + grid - 1) / grid;
  return ((r + kSRows - 1) / kSRows) * kSRows;
}

struct FinalMap {  // coarse bucket (+ next kRefBits key bits) -> final bucket
  const uint32_t* fbase;
  const uint8_t* gtab;
  const uint32_t* maxb;
  uint32_t cap;
  uint32_t spec_cap;   // speculative regions: spec_cap slots apart, `cap` usable (0: exact starts)
  uint32_t* spec_fail; // raised when a region overflows
  uint32_t* err;       // speculative mode: out-of-grid keys (the skipped histogram pass checks them)
  unsigned long long* bmp[2];  // level-L occupancy bits set here when non-null
};

template <bool NARROW>
__global__ void __launch_bounds__(kSThreads, 1)
    k_bkt_scatter(const double* __restrict__ src, const double* __restrict__ q,
                  const double* __restrict__ recv, const BucketGeo g, int level,
                  int64_t cta_rows, uint32_t* __restrict__ cursor, double* __restrict__ rec,
                  uint32_t* __restrict__ idx, const FinalMap fm) {
  extern __shared__ __align__(128) unsigned char sc_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sc_smem + (size_t)kSStages * kSStageBytes);
  uint64_t* empty = full + kSStages;
  const int tid = threadIdx.x;
  const int64_t n = g.n, tot = n + g.m;
  const int64_t lo = (int64_t)blockIdx.x * cta_rows;
  const int64_t hi = lo + cta_rows < tot ? lo + cta_rows : tot;
  if (lo >= hi) return;  // block-uniform
  const int nst = (int)((hi - lo + kSRows - 1) / kSRows);
  if (tid == 0) {
    for (int st = 0; st < kSStages; ++st) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + st)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + st)),
                   "r"(kSThreads));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t kmask = (1ull << g.sbits) - 1ull;
  const double grid = (double)(1ll << level);
  const bool refined = __ldg(fm.maxb) > fm.cap || wide_buckets(g);
  const int R = ref_bits(g);
  const bool qrec = g.qrec && q != nullptr;
  auto stage_xyz = [&](int k) {
    return reinterpret_cast<double*>(sc_smem + (size_t)(k % kSStages) * kSStageBytes);
  };
  auto stage_rows = [&](int k) {
    const int64_t base = lo + (int64_t)k * kSRows;
    return (int)(hi - base < kSRows ? hi - base : kSRows);
  };
  auto stage_tma = [&](int k) {
    const int64_t base = lo + (int64_t)k * kSRows;
    const int rows = stage_rows(k);
    const bool is_src = base < n;
    if (is_src && base + rows > n) return false;  // straddles src | recv
    const double* rp = row_ptr(src, recv, n, base);
    if (((uintptr_t)rp & 15) || ((rows * 24) & 15)) return false;
    if (is_src && qrec && (((uintptr_t)(q + base) & 15) || ((rows * 8) & 15))) return false;
    return true;
  };
  auto produce = [&](int k) {  // thread 0 only
    const int st = k % kSStages;
    if (k >= kSStages) mbar_wait(empty + st, (uint32_t)(k / kSStages - 1) & 1u);
    if (stage_tma(k)) {
      const int64_t base = lo + (int64_t)k * kSRows;
      const int rows = stage_rows(k);
      double* xyz = stage_xyz(k);
      const bool with_q = base < n && qrec;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(full + st, rows * 24 + (with_q ? rows * 8 : 0));
      bulk_g2s(xyz, row_ptr(src, recv, n, base), rows * 24, full + st);
      if (with_q) bulk_g2s(xyz + 3 * kSRows, q + base, rows * 8, full + st);
    } else {
      mbar_arrive(full + st);  // consumers fill this stage themselves
    }
  };
  // claim: wait for the stage, (fill it if it is a plain-load stage), slot atomic
  auto claim = [&](int k) -> uint32_t {
    const int st = k % kSStages;
    mbar_wait(full + st, (uint32_t)(k / kSStages) & 1u);
    double* xyz = stage_xyz(k);
    const int64_t i = lo + (int64_t)k * kSRows + tid;
    if (tid >= stage_rows(k)) return 0;
    if (!stage_tma(k)) {  // row-private fill: only this thread reads the row
      const double* p = row_ptr(src, recv, n, i);
      xyz[3 * tid] = __ldg(p);
      xyz[3 * tid + 1] = __ldg(p + 1);
      xyz[3 * tid + 2] = __ldg(p + 2);
      if (qrec && i < n) xyz[3 * kSRows + tid] = __ldg(q + i);
    }
    const uint64_t raw =
        encode_any<NARROW>(xyz[3 * tid], xyz[3 * tid + 1], xyz[3 * tid + 2], level, grid);
    if (fm.err && raw > kmask) atomicOr(fm.err, 1u);
    const uint64_t key = raw & kmask;
    if (fm.bmp[0]) {  // occupancy bit: fire-and-forget global reduction (no return)
      unsigned long long* w = fm.bmp[i >= n ? 1 : 0] + (key >> 6);
      asm volatile("red.global.or.b64 [%0], %1;" ::"l"(w), "l"(1ull << (key & 63)) : "memory");
    }
    uint32_t b = bucket_of(key, i >= n, g);
    if (refined)
      b = __ldg(fm.fbase + b) +
          __ldg(fm.gtab + (size_t)b * kRefBins + ((key >> (g.shift - R)) & ((1u << R) - 1u)));
    const uint32_t slot = atomicAdd(cursor + (size_t)b * kCursorStride, 1u);
    if (fm.spec_cap && slot - b * fm.spec_cap >= fm.cap) {  // region full
      atomicOr(fm.spec_fail, 1u);
      return 0xFFFFFFFFu;
    }
    return slot;
  };
  auto store = [&](int k, uint32_t dst) {
    const double* xyz = stage_xyz(k);
    const int64_t i = lo + (int64_t)k * kSRows + tid;
    if (tid < stage_rows(k) && dst != 0xFFFFFFFFu) {
      // record = {x, y, z, q} + the source index in the side array (qrec), or
      // {x, y, z, index within its set} (charges then follow the permutation
      // in k_gather_q): one 32-B store
      const bool sq = qrec && i < n;
      const double w = sq ? xyz[3 * kSRows + tid] : __longlong_as_double(i < n ? i : i - n);
      double x = xyz[3 * tid], y = xyz[3 * tid + 1], z = xyz[3 * tid + 2];
      const bool emb = sq && rec_embed(x, y, z, (uint32_t)i, g);  // index in the exponents
      st_v4f64(rec + 4 * (size_t)dst, x, y, z, w);
      if (sq && !emb) idx[dst] = (uint32_t)i;
    }
    mbar_arrive(empty + k % kSStages);
  };
  if (tid == 0)
    for (int k = 0; k < kSLead && k < nst; ++k) produce(k);
  // step k: produce k+lead, claim k, store k-depth; the slots of the last
  // depth+1 stages rotate through static registers (loop unrolled by depth+1)
  uint32_t d[kSDepth + 1] = {};
  auto step = [&](int k, uint32_t& dk, uint32_t dold) {
    if (tid == 0 && k + kSLead < nst) produce(k + kSLead);
    if (k < nst) dk = claim(k);
    if (k >= kSDepth && k - kSDepth < nst) store(k - kSDepth, dold);
  };
  for (int k = 0; k < nst + kSDepth; k += kSDepth + 1) {
#pragma unroll
    for (int j = 0; j <= kSDepth; ++j) step(k + j, d[j], d[(j + 1) % (kSDepth + 1)]);
  }
}

// ------------------------------------------------------------ local pass --
#ifndef FMMB_LCWARPS
#define FMMB_LCWARPS 8
#endif
constexpr int kLcWarps = FMMB_LCWARPS;
constexpr int kLcThreads = kLcWarps * 32;
constexpr int kLcDigit = 8;  // digit bits per in-smem LSD pass (fallback path)
constexpr int kLcBins = 1 << kLcDigit;
constexpr int kLcCap = 1280;  // points per bucket held in shared memory
constexpr int kLcSmallBits = 11;  // box-count path: <= 2^11 boxes per bucket
static_assert((1 << kLcSmallBits) <= kLcWarps * kLcBins, "box counters share s_wh");

template <typename CK>
__host__ __device__ constexpr size_t lc_smem_bytes() {
  // records | idx | composite x2 | slot x2 | per-warp digit counters | misc
  return (size_t)kLcCap * (32 + 4 + 2 * sizeof(CK) + 2 * 2) +
         (size_t)kLcWarps * kLcBins * 4 + 32 + 8 * kLcWarps + 64;
}

// One stable counting pass over digit [ds, ds+db) of B keys: warps own
// contiguous slices (ordered); per-warp digit counts by shared atomics, a
// digit-major scan over (digit, warp), then the placement walk ranks lanes
// with match.any so equal digits keep their order.
template <typename CK>
__device__ __forceinline__ void lc_pass(const CK* kin, const uint16_t* pin, CK* kout,
                                        uint16_t* pout, int B, int ds, int db,
                                        uint32_t* s_wh, uint32_t* s_red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbins = 1 << db;
  const uint32_t dm = (uint32_t)nbins - 1u;
  const int slice = ((B + kLcThreads - 1) / kLcThreads) * 32;
  const int lo = warp * slice;
  const int hi = lo + slice < B ? lo + slice : B;
  uint32_t* wh = s_wh + warp * kLcBins;
  for (int d = lane; d < nbins; d += 32) wh[d] = 0;
  __syncwarp();
  for (int j = lo + lane; j < hi; j += 32) atomicAdd(&wh[(uint32_t)(kin[j] >> ds) & dm], 1u);
  __syncthreads();
  // digit-major exclusive offsets: thread t owns digits [t*dpt, (t+1)*dpt)
  constexpr int dpt = (kLcBins + kLcThreads - 1) / kLcThreads;
  uint32_t tsum = 0;
#pragma unroll
  for (int e = 0; e < dpt; ++e) {
    const int d = threadIdx.x * dpt + e;
    if (d < nbins)
#pragma unroll
      for (int w = 0; w < kLcWarps; ++w) tsum += s_wh[w * kLcBins + d];
  }
  uint32_t wt;
  uint32_t x = warp_excl_scan(tsum, wt);
  if (lane == 0) s_red[warp] = wt;
  __syncthreads();
  for (int i = 0; i < warp; ++i) x += s_red[i];
#pragma unroll
  for (int e = 0; e < dpt; ++e) {
    const int d = threadIdx.x * dpt + e;
    if (d < nbins)
#pragma unroll
      for (int w = 0; w < kLcWarps; ++w) {
        const uint32_t c = s_wh[w * kLcBins + d];
        s_wh[w * kLcBins + d] = x;
        x += c;
      }
  }
  __syncthreads();
  const unsigned lt = lanemask_lt();
  for (int j0 = lo; j0 < hi; j0 += 32) {
    const int j = j0 + lane;
    CK k = 0;
    uint32_t d = 0xFFFFFFFFu;
    if (j < hi) {
      k = kin[j];
      d = (uint32_t)(k >> ds) & dm;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int leader = 31 - __clz(peers);  // highest lane of the group
    const uint32_t below = __popc(peers & lt);
    if (j < hi) {
      const uint32_t dst = wh[d] + below;
      kout[dst] = k;
      pout[dst] = pin[j];
    }
    __syncwarp();
    if (j < hi && lane == leader) wh[d] += below + 1;
    __syncwarp();
  }
  __syncthreads();
}

// One 24-byte point row with two stores: the 16-byte-aligned pair as one
// 16-byte store (x,y for an even row, y,z for an odd one) plus the other
// coordinate, instead of three 8-byte stores per row.
__device__ __forceinline__ void store_row(double* pts, int64_t p, double x, double y, double z) {
  // (explicit PTX: the two branch-wise equivalent forms must not be merged into
  // one unaligned 16-byte store)
  const bool odd = p & 1;
  double* row = pts + 3 * p;
  double* pair = row + (odd ? 1 : 0);
  double* one = row + (odd ? 0 : 2);
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(pair), "d"(odd ? y : x), "d"(odd ? z : y)
               : "memory");
  asm volatile("st.global.f64 [%0], %1;" ::"l"(one), "d"(odd ? x : z) : "memory");
}

struct LocalOut {
  double* pts;
  double* q;
  int64_t* perm;
  uint64_t* boxes;
  uint64_t* ne;
  int64_t* bm;
  unsigned long long* bmp[2];  // level-L occupancy bitmaps (may be null)
  int64_t* kinfo;
  const int64_t* gid[2];  // multi-GPU: global index of each local src / recv point (or null)
};

// permutation entry: local input index -> global index under the multi-GPU
// partition (identity for a single-GPU build)
__device__ __forceinline__ int64_t perm_of(const LocalOut& o, int set, int64_t local) {
  const int64_t* g = set ? o.gid[1] : o.gid[0];
  return g ? __ldg(g + local) : local;
}

// Ranking inside a bucket: with HEADS and <= 2^kLcSmallBits boxes per bucket,
// per-box counts (shared atomics), unstable placement into box segments and a
// rank of each point among its box's points by combined input index (boxes
// hold a handful of points; a box of more than 64 falls back).  Otherwise a
// LSD sort of the composite (low key bits, combined input index).
//
// HEADS: box heads go to the occupancy bitmap plus a bucket-local list of
// head positions (hpos[bs + h]); k_bkt_heads later writes bookmarks and
// non-empty keys at their global box ranks, taken from the bitmap's rank
// directory (no cross-bucket dependency here).  Without HEADS (sort_points:
// no bitmaps) the box ranks come from a decoupled look-back over buckets.
template <typename CK, bool NARROW, bool HEADS>
__global__ void __launch_bounds__(kLcThreads)
    k_bkt_local(const double* __restrict__ rec, uint32_t* __restrict__ idx,
                const uint32_t* __restrict__ bstart, const uint32_t* __restrict__ rbase,
                const BDesc* __restrict__ desc, const uint32_t* __restrict__ nfinal,
                const BucketGeo g, int level, const LocalOut o, uint64_t* __restrict__ states,
                const uint32_t* __restrict__ fail) {
  extern __shared__ __align__(128) unsigned char lc_smem[];
  double* s_rec = reinterpret_cast<double*>(lc_smem);                   // [cap][4]
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_rec + 4 * kLcCap);    // [cap]
  CK* k0 = reinterpret_cast<CK*>(s_idx + kLcCap);
  CK* k1 = k0 + kLcCap;
  uint16_t* p0 = reinterpret_cast<uint16_t*>(k1 + kLcCap);
  uint16_t* p1 = p0 + kLcCap;
  uint32_t* s_wh = reinterpret_cast<uint32_t*>(p1 + kLcCap);
  uint64_t* s_misc = reinterpret_cast<uint64_t*>(s_wh + kLcWarps * kLcBins);  // 16 B aligned
  uint32_t* s_red = reinterpret_cast<uint32_t*>(s_misc + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (__ldg(fail)) return;  // a final bucket overflows: the host reruns on the general path
  uint64_t* bar = s_misc + 2;
  const uint32_t nf = __ldg(nfinal);
  if (tid == 0) {
    mbar_init(bar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t bar_phase = 0;
  const int64_t n = g.n, m = g.m, tot = n + m;
  // persistent: every resident CTA walks the final buckets round-robin (in
  // order, so the non-HEADS look-back always finds its predecessors running).
  // (Double-buffering the records to prefetch the next bucket costs the third
  // resident CTA per SM and measured slower: 0.86 vs 0.69 ms at c2.)
  for (int64_t tile = blockIdx.x; tile < nf; tile += gridDim.x) {
  const int64_t bs = bstart[tile];  // output position of the bucket's first point
  const int B = (int)(bstart[tile + 1] - bs);
  const int64_t rb = rbase ? (int64_t)rbase[tile] : bs;  // its first record (speculative regions)
  const BDesc d = desc[tile];
  const int set = (int)(d.span_set >> 63);
  const uint64_t span = d.span_set & ~(1ull << 63);
  const uint64_t prefix = d.lo;  // first level-L key of the bucket; lk = key - lo
  if (B == 0) {  // empty final bucket: nothing to write (the look-back still needs its state)
    if (!HEADS && tid == 0) {
      uint64_t* st = states + tile;
      if (tile == 0) {
        st_state(st, kStInclusive);
      } else {
        st_state(st, kStAggregate);
        st_state(st, kStInclusive | lookback(states, tile, 0, 1));
      }
    }
    continue;
  }

  // phase 0: bulk copy of the bucket's records (TMA), source indices by LDG
  if (tid == 0) {
    const uint32_t bytes = (uint32_t)B * 32u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads
    mbar_expect_tx(bar, bytes);
    bulk_g2s(s_rec, rec + 4 * (size_t)rb, bytes, bar);
  }
  mbar_wait(bar, bar_phase);
  bar_phase ^= 1u;
  __syncthreads();
  // phase 1: low key bits and combined input index of every record; with
  // HEADS and <= 2^12 boxes per bucket also the per-box counts
  const double grid = (double)(1ll << level);
  const bool small = HEADS && span <= (1ull << kLcSmallBits);
  const int nbins = small ? (int)span : 1;
  if (small)
    for (int i = tid; i < nbins; i += kLcThreads) s_wh[i] = 0;
  __syncthreads();
  for (int j = tid; j < B; j += kLcThreads) {
    double* r = s_rec + 4 * j;
    // combined input index: embedded in a source record's exponents (the
    // coordinates are restored in place), else the idx side array (qrec),
    // else the record's last word (index within the set)
    uint32_t ci;
    if (g.qrec && set == 0) {
      if (!rec_extract(r, ci, g)) ci = __ldg(idx + rb + j);
    } else {
      ci = (uint32_t)(set ? n + __double_as_longlong(r[3]) : __double_as_longlong(r[3]));
    }
    const uint64_t key = encode_any<NARROW>(r[0], r[1], r[2], level, grid);
    // < span for every valid point; out-of-grid inputs (reported as a DomainError
    // after the build) are clamped so they cannot index outside the bucket
    uint64_t lk = (key & ((1ull << g.sbits) - 1ull)) - prefix;
    if (lk >= span) lk = 0;
    if (small) {
      k0[j] = (CK)lk;
      s_idx[j] = ci;
      atomicAdd(&s_wh[(uint32_t)lk], 1u);
    } else {
      k0[j] = ((CK)lk << g.cbits) | (CK)ci;
    }
    p0[j] = (uint16_t)j;
  }
  __syncthreads();
  bool ranked = false;
  if (small) {
    // per-box counts -> (count << 16 | start) cursors; heads straight from the
    // non-empty boxes; the largest box picks the ranking method
    constexpr int kBpt = (1 << kLcSmallBits) / kLcThreads;
    uint32_t c[kBpt];
    uint32_t csum = 0, nz = 0, cmax = 0;
#pragma unroll
    for (int e = 0; e < kBpt; ++e) {
      const int i = tid * kBpt + e;
      c[e] = i < nbins ? s_wh[i] : 0u;
      csum += c[e];
      nz += c[e] ? 1u : 0u;
      cmax = c[e] > cmax ? c[e] : cmax;
    }
    const uint32_t packed = (nz << 16) | csum;  // both < 2^16 per thread
    uint32_t wt;
    uint32_t x = warp_excl_scan(packed, wt);
    cmax = __reduce_max_sync(0xffffffffu, cmax);
    if (lane == 0) {
      s_red[warp] = wt;
      s_red[kLcWarps + warp] = cmax;
    }
    __syncthreads();
    uint32_t mx = 0;
    for (int i = 0; i < kLcWarps; ++i) {
      x += i < warp ? s_red[i] : 0u;
      mx = s_red[kLcWarps + i] > mx ? s_red[kLcWarps + i] : mx;
    }
    // every point is ranked inside its box by counting the smaller combined
    // indices of the box (O(box size) per point; a box of the whole bucket
    // costs kLcCap^2 / kLcThreads compares per thread, ~10 us): the LSD
    // fallback is never needed here, so CK only has to hold the composite
    // keys of the wide-bucket path (host: ck32)
    ranked = true;
    (void)mx;
    uint32_t start = x & 0xFFFFu, hidx = x >> 16;
    unsigned long long* bm = set ? o.bmp[1] : o.bmp[0];
    uint32_t* hp = idx + rb;
#pragma unroll
    for (int e = 0; e < kBpt; ++e) {
      const int i = tid * kBpt + e;
      if (i < nbins) {
        s_wh[i] = (c[e] << 16) | start;
        if (c[e]) {
          const uint64_t mk = prefix + (uint64_t)i;
          if (bm) atomicOr(bm + (mk >> 6), 1ull << (mk & 63));
          hp[hidx] = (uint32_t)(bs + start - (set ? n : 0));
          ++hidx;
        }
      }
      start += c[e];
    }
    __syncthreads();
    if (!ranked) {  // a crowded box: fall back to the LSD passes below
      for (int j = tid; j < B; j += kLcThreads)
        k0[j] = ((CK)k0[j] << g.cbits) | (CK)s_idx[j];
      __syncthreads();
    }
  }
  if (ranked) {
    // unstable placement into box segments, then rank inside the box by the
    // combined input index (unique): position = start + #smaller indices
    CK* tci = k1;
    uint16_t* tj = p1;
    for (int j = tid; j < B; j += kLcThreads) {
      const uint32_t slot = atomicAdd(&s_wh[(uint32_t)k0[j]], 1u) & 0xFFFFu;
      tci[slot] = (CK)s_idx[j];
      tj[slot] = (uint16_t)j;
    }
    __syncthreads();
    for (int t = tid; t < B; t += kLcThreads) {
      const uint32_t ci = (uint32_t)tci[t];
      const int j = tj[t];
      const uint32_t v = s_wh[(uint32_t)k0[j]];
      const uint32_t end = v & 0xFFFFu, cnt = v >> 16;
      uint32_t rank = 0;
#pragma unroll 4
      for (uint32_t u = end - cnt; u < end; ++u) rank += (uint32_t)tci[u] < ci ? 1u : 0u;
      p0[end - cnt + rank] = (uint16_t)j;
    }
    __syncthreads();
    // phase 4 (ranked): outputs in sorted order; heads were written above
    for (int pos = tid; pos < B; pos += kLcThreads) {
      const int64_t p = bs + pos;
      const int j = p0[pos];
      const double* r = s_rec + 4 * j;
      store_row(o.pts, p, r[0], r[1], r[2]);
      o.perm[p] = perm_of(o, set, (int64_t)s_idx[j] - (set ? n : 0));
      if (g.qrec && set == 0 && o.q) o.q[p] = r[3];
      o.boxes[p] = prefix + (uint64_t)k0[j];
    }
    __syncthreads();  // smem reused by the next bucket
    continue;
  }
  // phase 2: LSD passes over the composite (index bits first, then key bits)
  CK* kc = k0;
  uint16_t* pc = p0;
  int lbits = 0;
  while (lbits < 63 && (1ull << lbits) < span) ++lbits;
  const int cbits = lbits + g.cbits;
  for (int ds = 0; ds < cbits; ds += kLcDigit) {
    const int db = cbits - ds < kLcDigit ? cbits - ds : kLcDigit;
    CK* ko = kc == k0 ? k1 : k0;
    uint16_t* po = pc == p0 ? p1 : p0;
    lc_pass<CK>(kc, pc, ko, po, B, ds, db, s_wh, s_red);
    kc = ko;
    pc = po;
  }
  const int wb = g.cbits;
  int64_t hbase = 0;
  if (!HEADS) {
    // phase 3: head count, box-rank base by look-back over buckets
    uint32_t hc = 0;
    for (int j = tid; j < B; j += kLcThreads)
      hc += (j == 0 || (kc[j] >> wb) != (kc[j - 1] >> wb)) ? 1u : 0u;
    hc = __reduce_add_sync(0xffffffffu, hc);
    if (lane == 0) s_red[warp] = hc;
    __syncthreads();
    if (tid == 0) {
      uint32_t heads = 0;
      for (int i = 0; i < kLcWarps; ++i) heads += s_red[i];
      uint64_t* st = states + tile;
      uint64_t excl = 0;
      if (tile == 0) {
        st_state(st, kStInclusive | heads);
      } else {
        st_state(st, kStAggregate | heads);
        excl = lookback(states, tile, 0, 1);
        st_state(st, kStInclusive | (excl + heads));
      }
      s_misc[1] = excl;
    }
    __syncthreads();
    hbase = (int64_t)s_misc[1];
  }
  unsigned long long* bmp = set ? o.bmp[1] : o.bmp[0];
  uint32_t* hpos = idx + rb;  // HEADS: this bucket's idx slots are free again
  const unsigned lt = lanemask_lt();
  // phase 4: outputs in sorted order (chunks of kLcThreads, scan of heads)
  for (int j0 = 0; j0 < B; j0 += kLcThreads) {
    const int j = j0 + tid;
    const bool ok = j < B;
    bool head = false;
    uint64_t lk = 0;
    if (ok) {
      lk = (uint64_t)(kc[j] >> wb);
      head = j == 0 || (uint64_t)(kc[j - 1] >> wb) != lk;
    }
    const unsigned hb = __ballot_sync(0xffffffffu, head);
    if (lane == 0) s_red[kLcWarps + warp] = __popc(hb);
    __syncthreads();
    uint32_t woff = 0, ctot = 0;
#pragma unroll
    for (int i = 0; i < kLcWarps; ++i) {
      const uint32_t c = s_red[kLcWarps + i];
      woff += i < warp ? c : 0u;
      ctot += c;
    }
    if (ok) {
      const int64_t p = bs + j;  // combined sorted position
      const int pl = pc[j];
      const double* r = s_rec + 4 * pl;
      const uint64_t mk = prefix + lk;
      store_row(o.pts, p, r[0], r[1], r[2]);
      const int64_t ci = (int64_t)((uint64_t)kc[j] & ((1ull << wb) - 1ull));  // combined index
      o.perm[p] = perm_of(o, set, ci - (set ? n : 0));
      if (g.qrec && set == 0 && o.q) o.q[p] = r[3];
      o.boxes[p] = mk;
      const int64_t incl = hbase + woff + __popc(hb & (lt | (1u << lane)));
      if (head) {
        if (bmp) atomicOr(bmp + (mk >> 6), 1ull << (mk & 63));
        if (HEADS) {
          hpos[incl - 1] = (uint32_t)(p - (set ? n : 0));
        } else {
          const int64_t jg = incl - 1;
          o.ne[jg] = mk;
          o.bm[jg + set] = p - (set ? n : 0);
        }
      }
      if (!HEADS) {
        if (p == n - 1) {
          o.kinfo[0] = incl;
          o.bm[incl] = n;
          if (m == 0) o.bm[incl + 1] = 0;
        }
        if (p == tot - 1 && m > 0) {
          o.kinfo[1] = incl;
          o.bm[incl + 1] = m;
          if (n == 0) {
            o.bm[0] = 0;
            o.kinfo[0] = 0;
          }
        }
      }
    }
    hbase += ctot;
    __syncthreads();  // s_red[8..] reused by the next chunk
  }
  }  // final buckets
}

// sorted charges: q_out[p] = q[perm[p]] for the n source positions (the
// bucket records carry the index, not the charge); four independent
// gathers in flight per thread.  Runs before k_gid_map (perm is still the
// local index then).
__global__ void __launch_bounds__(256)
    k_gather_q(const int64_t* __restrict__ perm, const double* __restrict__ q, int64_t n,
               double* __restrict__ q_out, const uint32_t* __restrict__ fail) {
  if (__ldg(fail)) return;  // the sort reruns on the general path
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x * 4 + threadIdx.x; b < n; b += stride) {
    int64_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t p = b + (int64_t)k * blockDim.x;
      v[k] = p < n ? __ldcs(perm + p) : 0;
    }
    double w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t p = b + (int64_t)k * blockDim.x;
      w[k] = p < n ? __ldg(q + v[k]) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t p = b + (int64_t)k * blockDim.x;
      if (p < n) __stcs(q_out + p, w[k]);
    }
  }
}

// perm[p] = gid[perm[p]] of its set (multi-GPU: local -> global input index);
// four independent gathers in flight per thread
__global__ void __launch_bounds__(256)
    k_gid_map(int64_t* __restrict__ perm, int64_t n, int64_t m, const int64_t* __restrict__ g0,
              const int64_t* __restrict__ g1, const uint32_t* __restrict__ fail) {
  if (__ldg(fail)) return;  // the sort reruns on the general path
  const int64_t tot = n + m;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x * 4 + threadIdx.x; b < tot; b += stride) {
    int64_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t p = b + (int64_t)k * blockDim.x;
      v[k] = p < tot ? perm[p] : 0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t p = b + (int64_t)k * blockDim.x;
      if (p < tot) {
        const int64_t* g = p < n ? g0 : g1;
        v[k] = g ? __ldg(g + v[k]) : v[k];
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t p = b + (int64_t)k * blockDim.x;
      if (p < tot) perm[p] = v[k];
    }
  }
}

// Bookmarks and non-empty keys at their global box ranks (HEADS variant):
// one warp per bucket walks the bucket's words of the level-L bitmap; the
// h-th set bit is the bucket's h-th box, its rank = rank directory + prefix
// popcount, its first point = hpos[bs + h].
struct HeadsParams {
  const uint64_t* bmp[2];  // level-L bitmaps (src, recv)
  const uint32_t* dir[2];  // their rank directories
  const int64_t* ktot_src;  // K_s (device, from k_rank)
  const int64_t* ktot_recv; // K_r
  const uint32_t* bstart;
  const uint32_t* rbase;  // record / hpos base per final bucket (null: = bstart)
  const uint32_t* hpos;
  uint64_t* ne;
  int64_t* bm;
  int64_t* kinfo;
};

__global__ void __launch_bounds__(256)
    k_bkt_heads(const __grid_constant__ HeadsParams hp, const BDesc* __restrict__ desc,
                const uint32_t* __restrict__ nfinal, const BucketGeo g) {
  const int lane = threadIdx.x & 31;
  const int64_t ks = *hp.ktot_src;
  const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (gw == 0 && lane == 0) {
    const int64_t kr = *hp.ktot_recv;
    hp.bm[ks] = g.n;
    hp.bm[ks + 1 + kr] = g.m;
    hp.kinfo[0] = ks;
    hp.kinfo[1] = ks + kr;
  }
  const uint32_t nf = __ldg(nfinal);
  const unsigned lt = lanemask_lt();
  for (int64_t f = gw; f < nf; f += (int64_t)gridDim.x * 8) {
    if (hp.bstart[f + 1] == hp.bstart[f]) continue;  // empty final bucket
    const BDesc d = desc[f];
    const int set = (int)(d.span_set >> 63);
    const uint64_t nbits = d.span_set & ~(1ull << 63);
    const uint64_t key0 = d.lo;
    const uint64_t* bmp = set ? hp.bmp[1] : hp.bmp[0];
    const uint32_t* dir = set ? hp.dir[1] : hp.dir[0];
    const uint32_t* hpos = hp.hpos + (hp.rbase ? hp.rbase[f] : hp.bstart[f]);
    uint64_t* ne = hp.ne + (set ? ks : 0);
    int64_t* bm = hp.bm + (set ? ks + 1 : 0);
    const int64_t w0 = (int64_t)(key0 >> 6);
    const uint64_t below0 = (key0 & 63) ? (__ldg(bmp + w0) & ((1ull << (key0 & 63)) - 1ull)) : 0ull;
    const int64_t rank0 = (int64_t)__ldg(dir + w0) + __popcll(below0);
    int64_t h = 0;
    // lane = box: 32 consecutive keys per step; all-zero 64-bit words skipped
    for (uint64_t off = 0; off < nbits; off += 32) {
      const uint64_t key = key0 + off + lane;
      const uint64_t word = __ldg(bmp + (key >> 6));
      if (__all_sync(0xffffffffu, word == 0)) {  // skip the rest of an empty word
        off = ((key0 + off + 64) & ~63ull) - key0 - 32;
        continue;
      }
      const bool occ = off + lane < nbits && ((word >> (key & 63)) & 1ull);
      const unsigned ballot = __ballot_sync(0xffffffffu, occ);
      if (occ) {
        const int64_t at = h + __popc(ballot & lt);
        ne[rank0 + at] = key;
        bm[rank0 + at] = (int64_t)__ldg(hpos + at);
      }
      h += __popc(ballot);
    }
  }
}

}  // namespace fmmb
