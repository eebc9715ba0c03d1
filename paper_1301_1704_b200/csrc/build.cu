// libfmmb200: C-ABI entry points for the fused build (fmmb_build_all,
// fmmb_sort_points) and the handle lifecycle.  Host orchestration of the
// sm_100a kernels in sort.cuh / finalize.cuh / lists.cuh.
//
// build_all (reference lists.py:133-187) runs as two stream-ordered phases:
//   A: encode+histogram -> P radix passes -> gather/bookmarks/bitmap_L ->
//      bitmap pyramid -> rank directory + level directory -> list counts ->
//      segmented scan into the CSR bookmarks
//   -- one device->host read of the sizes (K per level, |E2|, |E4_l|) --
//   B: list write pass into exactly-sized outputs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <functional>
#include <vector>

#include "internal.h"
#include "common.cuh"
#include "bucket.cuh"
#include "dist.cuh"
#include "finalize.cuh"
#include "lists.cuh"
#include "sort.cuh"

using namespace fmmb;

// ------------------------------------------------------------------ handle
// error text of the calling thread's last failed call (thread-local, so a
// concurrent caller cannot overwrite it between the failure and the read)
static thread_local std::string t_err;

fmmb_status fmmb_fail(fmmb_handle_t h, fmmb_status st, const char* fmt, ...) {
  (void)h;
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_err = buf;
  return st;
}

extern "C" int fmmb_abi_version(void) { return FMMB_ABI_VERSION; }

extern "C" fmmb_status fmmb_create(int device, fmmb_handle_t* out) {
  if (!out) return FMMB_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return FMMB_ERR_CUDA;
  auto* h = new fmmb_handle_s();
  h->device = device;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    delete h;
    return FMMB_ERR_CUDA;
  }
  h->num_sms = prop.multiProcessorCount;
  h->pinned = nullptr;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaMallocHost(&h->pinned, kPinnedBytes) != cudaSuccess) {
    delete h;
    return FMMB_ERR_CUDA;
  }
  {
    cudaStream_t side, side_hi;
    cudaEvent_t e[6];
    // two sort streams: default priority (late occupancy: the local pass
    // beside the lists) and the highest priority (early occupancy: the sort
    // chain is the critical path, its pending CTAs go first -- c3 3.17 vs
    // 3.41 ms; c2/c4 are better without); FMMB_SIDE_PRIO=1: always high
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    const char* sp = getenv("FMMB_SIDE_PRIO");
    const int prio = (sp && atoi(sp)) ? hi_prio : 0;
    if (cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, prio) != cudaSuccess ||
        cudaStreamCreateWithPriority(&side_hi, cudaStreamNonBlocking, hi_prio) != cudaSuccess) {
      cudaFreeHost(h->pinned);
      delete h;
      return FMMB_ERR_CUDA;
    }
    h->side_hi = side_hi;
    for (auto& x : e) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    h->side = side;
    h->ev_split = e[0];
    h->ev_rank = e[1];
    h->ev_side = e[2];
    h->ev_plan = e[3];
    h->ev_count = e[4];
    h->ev_rb = e[5];
    h->lists_upfront = getenv("FMMB_LISTS_EXACT") == nullptr;
    // early occupancy: the scatter right after the refinement plan (c3 3.16 vs
    // 3.43 ms with it waiting for the list count); FMMB_SCATTER_AFTER_COUNT=1
    h->scatter_after_count = getenv("FMMB_SCATTER_AFTER_COUNT") != nullptr;
    h->overlap = getenv("FMMB_NO_OVERLAP") == nullptr;
    h->early_occ = getenv("FMMB_LATE_OCC") ? 0 : getenv("FMMB_EARLY_OCC") ? 2 : 1;
    h->rec_q = getenv("FMMB_REC_IDX") == nullptr;
    h->rec_embed = getenv("FMMB_NO_EMBED") == nullptr;
    const char* sc = getenv("FMMB_SCATTER_CTAS");
    h->scatter_ctas = sc ? atoi(sc) : 0;
    h->trace = getenv("FMMB_TRACE") != nullptr;
    if (h->trace)
      for (auto& x : h->tr_ev) cudaEventCreate((cudaEvent_t*)&x);
    h->local_after_count = getenv("FMMB_LOCAL_AFTER") != nullptr;
    const char* lc = getenv("FMMB_LC_PER_SM");
    h->lc_per_sm = lc ? atoi(lc) : 0;
    const char* csp = getenv("FMMB_CS_PER_SM");  // persistent list-count grid (A/B)
    h->cs_per_sm = csp ? atoi(csp) : 0;
    const char* lw = getenv("FMMB_LW_PER_SM");  // list-write CTAs per SM in the grid (A/B)
    h->lw_per_sm = lw ? std::max(1, atoi(lw)) : 32;
    h->dense_rows = getenv("FMMB_DENSE_ROWS") != nullptr;
  }
  // stream-ordered pool: keep freed workspace for reuse across calls
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  // opt-in dynamic shared memory for the big-tile kernels
  cudaFuncSetAttribute(k_onesweep<uint32_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)onesweep_smem_bytes(4));
  cudaFuncSetAttribute(k_onesweep<uint32_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)onesweep_smem_bytes(4));
  cudaFuncSetAttribute(k_onesweep<uint64_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)onesweep_smem_bytes(8));
  cudaFuncSetAttribute(k_onesweep<uint64_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)onesweep_smem_bytes(8));
  cudaFuncSetAttribute(k_bkt_hist<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (2 << kBucketBitsMax) * (int)sizeof(uint32_t));
  cudaFuncSetAttribute(k_bkt_hist<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (2 << kBucketBitsMax) * (int)sizeof(uint32_t));
  cudaFuncSetAttribute(k_bkt_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)scatter_smem_bytes());
  cudaFuncSetAttribute(k_bkt_scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)scatter_smem_bytes());
  cudaFuncSetAttribute(k_part_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(uint32_t) << kPartMaxBits));
#define FMMB_LCATTR(CK, NW, HD)                                                        \
  cudaFuncSetAttribute(k_bkt_local<CK, NW, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                       (int)lc_smem_bytes<CK>())
  FMMB_LCATTR(uint32_t, true, true);
  FMMB_LCATTR(uint32_t, true, false);
  FMMB_LCATTR(uint32_t, false, true);
  FMMB_LCATTR(uint32_t, false, false);
  FMMB_LCATTR(uint64_t, true, true);
  FMMB_LCATTR(uint64_t, true, false);
  FMMB_LCATTR(uint64_t, false, true);
  FMMB_LCATTR(uint64_t, false, false);
#undef FMMB_LCATTR
  cudaFuncSetAttribute(k_gather<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)gather_smem_bytes());
  cudaFuncSetAttribute(k_gather<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)gather_smem_bytes());
  if (cudaGetLastError() != cudaSuccess) {
    cudaFreeHost(h->pinned);
    delete h;
    return FMMB_ERR_CUDA;
  }
  *out = h;
  return FMMB_OK;
}

extern "C" fmmb_status fmmb_destroy(fmmb_handle_t h) {
  if (!h) return FMMB_ERR_ARG;
  cudaSetDevice(h->device);
  if (h->pinned) cudaFreeHost(h->pinned);
  if (h->side) cudaStreamDestroy((cudaStream_t)h->side);
  if (h->side_hi) cudaStreamDestroy((cudaStream_t)h->side_hi);
  for (void* e : {h->ev_split, h->ev_rank, h->ev_side, h->ev_plan, h->ev_count, h->ev_rb})
    if (e) cudaEventDestroy((cudaEvent_t)e);
  for (void* e : h->tr_ev)
    if (e) cudaEventDestroy((cudaEvent_t)e);
  delete h;
  return FMMB_OK;
}

extern "C" const char* fmmb_last_error(fmmb_handle_t h) {
  return h ? t_err.c_str() : "null handle";
}

extern "C" int64_t fmmb_last_launch_count(fmmb_handle_t h) { return h ? h->launches : -1; }

void fmmb_trace_point(fmmb_handle_t h, const char* name, void* stream) {
  if (!h->trace || h->tr_n >= 32) return;
  cudaEventRecord((cudaEvent_t)h->tr_ev[h->tr_n], (cudaStream_t)stream);
  h->tr_name[h->tr_n++] = name;
}

extern "C" int fmmb_trace(fmmb_handle_t h, float* ms, const char** names, int cap) {
  if (!h || !h->trace) return 0;
  FMMB_GUARD(h);
  const int k = std::min(cap, h->tr_n);
  for (int i = 0; i < k; ++i) {
    cudaEventSynchronize((cudaEvent_t)h->tr_ev[i]);
    float t = 0.f;
    cudaEventElapsedTime(&t, (cudaEvent_t)h->tr_ev[0], (cudaEvent_t)h->tr_ev[i]);
    ms[i] = t;
    names[i] = h->tr_name[i];
  }
  return k;
}

extern "C" fmmb_status fmmb_set_sort_path(fmmb_handle_t h, int path) {
  FMMB_GUARD(h);
  if (!h || path < 0 || path > 3) return FMMB_ERR_ARG;
  h->sort_path = path;
  return FMMB_OK;
}

extern "C" int fmmb_last_sort_path(fmmb_handle_t h) { return h ? h->last_sort_path : -1; }

extern "C" fmmb_status fmmb_set_overlap(fmmb_handle_t h, int on) {
  FMMB_GUARD(h);
  if (!h) return FMMB_ERR_ARG;
  h->overlap = on != 0;
  return FMMB_OK;
}

int lists_lmin_host(int L) { return L >= 2 ? 2 : L; }

// --------------------------------------------------------------- arenas --
namespace {

struct Carver {  // sub-allocates 256-B aligned slices of one allocation
  size_t off = 0;
  template <typename T>
  size_t take(int64_t count) {
    const size_t at = off;
    off += ((size_t)std::max<int64_t>(count, 0) * sizeof(T) + 255) & ~(size_t)255;
    return at;
  }
};

inline int64_t cap_level(int64_t count, int level) {  // min(count, 8^level)
  if (3 * level >= 62) return count;
  return std::min<int64_t>(count, 1ll << (3 * level));
}

inline int64_t level_words(int level) {  // u64 words of a level bitmap
  const int64_t bits = 1ll << (3 * level);
  return std::max<int64_t>(1, bits / 64);
}

}  // namespace

// Bitmap path limit: the level-L occupancy bitmap of one set is 8^L/8 bytes.
bool fmmb_bitmap_ok(int level, int64_t n_total) {
  if (level > 12) return false;
  const double bytes = std::ldexp(1.0, 3 * level) / 8.0;
  return bytes <= std::max(64.0 * 1024 * 1024, 4.0 * 8.0 * (double)n_total);
}

// --------------------------------------------------------------- build ---
namespace {

struct BuildPlanHost {  // mirrored in the pinned readback block
  int64_t ktot[kMaxSegs];
  int64_t seg_totals[kMaxLevel + 1];
  int64_t kinfo[2];
  uint32_t err;
  uint32_t fail;       // bucket path overflowed its shared-memory capacity
  uint32_t spec_fail;  // a speculative bucket region overflowed
};

// ---- sort phase, fast path: payload-carrying bucket sort (bucket.cuh)
struct BucketRun {  // scratch that outlives the sort phase (heads pass)
  std::function<void(cudaStream_t)> local;  // the local pass (+ gid map), launched by the caller
  std::function<void(cudaStream_t)> scatter;  // deferred scatter (early occupancy), or empty
  char* scratch = nullptr;
  BucketGeo g{};
  const uint32_t* bstart_f = nullptr;
  const uint32_t* rbase = nullptr;
  const BDesc* desc = nullptr;
  const uint32_t* nfinal = nullptr;
  const uint32_t* hpos = nullptr;
};

template <typename CK, bool NARROW, bool HEADS>
void launch_local(fmmb_handle_t h, const double* rec, uint32_t* idx, const uint32_t* bstart_f,
                  const uint32_t* rbase, const BDesc* desc, const uint32_t* nfinal,
                  const BucketGeo& g, int L, const LocalOut& o, uint64_t* lst,
                  const uint32_t* fail, int cap, cudaStream_t s) {
  auto kern = k_bkt_local<CK, NARROW, HEADS>;
  static const int occ = [&] {  // resident CTAs per SM (same on every B200), once
    int v = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, kLcThreads, lc_smem_bytes<CK>());
    return v;
  }();
  int per_sm = occ;
  if (h->lc_per_sm > 0) cap = h->lc_per_sm;
  if (cap > 0) per_sm = std::min(per_sm, cap);
  const int grid = std::max(1, per_sm) * h->num_sms;  // persistent: all CTAs resident
  kern<<<grid, kLcThreads, lc_smem_bytes<CK>(), s>>>(rec, idx, bstart_f, rbase, desc, nfinal, g,
                                                     L, o, lst, fail);
}

template <bool NARROW>
void launch_spec(const double* src, const double* q, const double* recv, const BucketGeo& g,
                 int num_sms, int L, uint32_t* counts, uint32_t* bstart, uint64_t* sst,
                 uint32_t* ctl, uint32_t* rbase, const PlanOut& po, double* rec, uint32_t* idx,
                 uint32_t* spec_fail, uint32_t* err, cudaStream_t s,
                 unsigned long long* const* sbmp, std::function<void(cudaStream_t)>* tail) {
  const unsigned nbg = (unsigned)ceil_div(g.nb, 256);
  k_spec_init<<<nbg, 256, 0, s>>>(g, kSpecStride, po.cursor, rbase, po.desc, po.nfinal);
  const int sgrid = (int)std::min<int64_t>(num_sms, ceil_div(g.n + g.m, kSRows));
  FinalMap fm{po.fbase, po.gtab, ctl + 4, kLcCap, (uint32_t)kSpecStride, spec_fail, err,
              {nullptr, nullptr}};
  fm.bmp[0] = sbmp[0];
  fm.bmp[1] = sbmp[1];
  k_bkt_scatter<NARROW><<<(unsigned)sgrid, kSThreads, scatter_smem_bytes(), s>>>(
      src, q, recv, g, L, scatter_rows_per_cta(g.n + g.m, sgrid), po.cursor, rec, idx, fm);
  // bucket starts from the final cursors: only the local pass and the heads
  // need them, so they run on the local pass's stream (the directory starts
  // right after the scatter)
  BucketGeo g1 = g;
  g1.hgrid = 1;
  uint32_t* cursor = po.cursor;
  *tail = [=](cudaStream_t st) {
    k_spec_counts<<<nbg, 256, 0, st>>>(g, kSpecStride, cursor, counts);
    k_bkt_scan<<<(unsigned)ceil_div(g.nb, kScanBuckets), 256, 0, st>>>(counts, g1, bstart, sst,
                                                                       ctl + 0, ctl + 2);
  };
}

// Histogram path.  With `early` the histogram pass (on `s`) also sets the
// level-L occupancy bits and everything after it (scan, refinement plan,
// scatter) goes to the sort stream `ss`, split off by ev_split: the caller's
// stream continues with the directory and the lists while the sort runs.
// ev_plan (when non-null) marks the plan on `ss`: the refinement overflow
// flag is final there, long before the scatter ends.
template <bool NARROW>
void launch_hs(const double* src, const double* q, const double* recv, const BucketGeo& g,
               int num_sms, int L, uint32_t* mat, uint32_t* bstart, uint64_t* sst, uint32_t* ctl,
               uint32_t* fine, const PlanOut& po, double* rec, uint32_t* idx, uint32_t* err,
               cudaStream_t s, unsigned long long* const* sbmp, bool early, cudaStream_t ss,
               cudaEvent_t ev_split, cudaEvent_t ev_plan, int scatter_ctas,
               std::function<void(cudaStream_t)>* defer_scatter) {
  const bool wide = g.shift > kLcSmallBits;  // every non-empty bucket is refined
  k_bkt_hist<NARROW><<<(unsigned)g.hgrid, kHThreads, (size_t)g.nb * 4, s>>>(
      src, recv, g, L, mat, err, wide ? fine : nullptr, early ? sbmp[0] : nullptr,
      early ? sbmp[1] : nullptr);
  if (early && ss != s) {
    cudaEventRecord(ev_split, s);
    cudaStreamWaitEvent(ss, ev_split, 0);
  } else {
    ss = s;
  }
  k_bkt_scan<<<(unsigned)ceil_div(g.nb, kScanBuckets), 256, 0, ss>>>(mat, g, bstart, sst,
                                                                     ctl + 0, ctl + 2);
  if (!wide)
    k_bkt_fine<NARROW><<<num_sms * 8, 256, 0, ss>>>(src, recv, g, L, bstart, ctl + 2, kLcCap,
                                                    fine);
  k_bkt_plan<<<(unsigned)ceil_div(g.nb, 256), 256, 0, ss>>>(g, bstart, ctl + 2, kLcCap, fine, po);
  if (ev_plan) cudaEventRecord(ev_plan, ss);
  const int sgrid = (int)std::min<int64_t>(std::min(num_sms, std::max(1, scatter_ctas)),
                                           ceil_div(g.n + g.m, kSRows));
  const FinalMap fm{po.fbase, po.gtab, ctl + 2, kLcCap, 0u, nullptr, nullptr,
                    {early ? nullptr : sbmp[0], early ? nullptr : sbmp[1]}};
  const int64_t rows = scatter_rows_per_cta(g.n + g.m, sgrid);
  uint32_t* cursor = po.cursor;
  auto scatter = [=](cudaStream_t st) {
    k_bkt_scatter<NARROW><<<(unsigned)sgrid, kSThreads, scatter_smem_bytes(), st>>>(
        src, q, recv, g, L, rows, cursor, rec, idx, fm);
  };
  if (defer_scatter) *defer_scatter = scatter;  // launched by the caller (after the list count)
  else scatter(ss);
}

// speculative regions apply when the coarse buckets already fit the count path
inline bool spec_possible(const BucketGeo& g) { return g.shift <= kLcSmallBits; }

// the local pass's LSD fallback sorts (in-bucket key bits, combined index) as
// one 64-bit composite: every final bucket's key span plus the index bits
// must fit, else the build takes the Onesweep path (L = 20 with ~2^28
// points).  Wide coarse buckets are always refined along kRefBits more key
// bits (k_bkt_plan: one sub-bin per final bucket once the sub-bins span
// >= 2^kLcSmallBits keys).
inline int final_span_bits(const BucketGeo& g) {
  return g.shift > kLcSmallBits ? std::max(g.shift - kRefBits, kLcSmallBits) : g.shift;
}
inline bool bucket_fits(const BucketGeo& g) { return final_span_bits(g) + g.cbits <= 64; }

fmmb_status sort_bucket(fmmb_handle_t h, const double* src, const double* q, int64_t n,
                        const double* recv, int64_t m, int L, const LocalOut& o, bool heads,
                        bool spec, BuildPlanHost* dplan, cudaStream_t s, int64_t& launches,
                        BucketRun& run, cudaStream_t ls, bool early) {
  BucketGeo g = bucket_geo(L, n, m, h->num_sms);
  g.qrec = (q && n > 0 && h->rec_q) ? 1 : 0;
  // index embedding in the source records' exponents: 34 payload bits hold
  // the index and three exponents of eb bits (FMMB_NO_EMBED=1: side store only)
  g.eb = (g.qrec && h->rec_embed) ? std::min(3, (34 - g.cbits) / 3) : 0;
  if (g.eb < 1) g.eb = 0;
  const int64_t tot = n + m;
  const int64_t nfcap = final_buckets_cap(g, kLcCap);
  const int64_t nrec = spec ? (int64_t)g.nb * kSpecStride : tot;  // record slots
  Carver c;
  const size_t o_sst = c.take<uint64_t>(ceil_div(g.nb, kScanBuckets));
  const size_t o_pst = c.take<uint64_t>(ceil_div(g.nb, 256));
  const size_t o_lst = c.take<uint64_t>(nfcap);
  const size_t o_ctl = c.take<uint32_t>(8);  // [0] scan ticket, [1] plan ticket, [2] max bucket, [3] nfinal, [4] zero
  const size_t o_fine = c.take<uint32_t>((int64_t)g.nb * kRefBins);
  const size_t o_gtab = c.take<uint8_t>((int64_t)g.nb * kRefBins);
  const size_t zero_bytes = c.off;
  const size_t o_mat = c.take<uint32_t>((int64_t)g.hgrid * g.nb);
  const size_t o_bs = c.take<uint32_t>(g.nb + 1);
  const size_t o_fb = c.take<uint32_t>(g.nb);
  const size_t o_bsf = c.take<uint32_t>(nfcap + 1);
  const size_t o_desc = c.take<BDesc>(nfcap);
  const size_t o_cur = c.take<uint32_t>(nfcap * kCursorStride);
  const size_t o_rec = c.take<double>(4 * nrec);
  const size_t o_idx = c.take<uint32_t>(nrec);
  const size_t o_rb = c.take<uint32_t>(spec ? g.nb : 0);
  char* w = nullptr;
  if (cudaMallocAsync((void**)&w, c.off, s) != cudaSuccess)
    return fmmb_fail(h, FMMB_ERR_CUDA, "bucket-sort scratch of %zu bytes failed", c.off);
  cudaMemsetAsync(w, 0, zero_bytes, s);
  uint32_t* ctl = (uint32_t*)(w + o_ctl);
  uint32_t* mat = (uint32_t*)(w + o_mat);
  uint32_t* bstart = (uint32_t*)(w + o_bs);
  double* rec = (double*)(w + o_rec);
  uint32_t* idx = (uint32_t*)(w + o_idx);
  uint64_t* sst = (uint64_t*)(w + o_sst);
  uint64_t* lst = (uint64_t*)(w + o_lst);
  PlanOut po{};
  po.fbase = (uint32_t*)(w + o_fb);
  po.gtab = (uint8_t*)(w + o_gtab);
  po.bstart_f = (uint32_t*)(w + o_bsf);
  po.desc = (BDesc*)(w + o_desc);
  po.cursor = (uint32_t*)(w + o_cur);
  po.nfinal = ctl + 3;
  po.fail = &dplan->fail;
  po.states = (uint64_t*)(w + o_pst);
  po.ticket = ctl + 1;
  uint32_t* fine = (uint32_t*)(w + o_fine);
  const bool narrow = L <= 10;
  uint32_t* rbase = spec ? (uint32_t*)(w + o_rb) : nullptr;
  std::function<void(cudaStream_t)> spec_tail;  // spec path: bucket starts, before the local pass
  if (spec) {  // no histogram pass: fixed regions, exact starts from the final cursors
    if (narrow)
      launch_spec<true>(src, q, recv, g, h->num_sms, L, mat, bstart, sst, ctl, rbase, po, rec,
                        idx, &dplan->spec_fail, &dplan->err, s, o.bmp, &spec_tail);
    else
      launch_spec<false>(src, q, recv, g, h->num_sms, L, mat, bstart, sst, ctl, rbase, po, rec,
                         idx, &dplan->spec_fail, &dplan->err, s, o.bmp, &spec_tail);
    po.bstart_f = bstart;
  } else {
    cudaEvent_t evs = (cudaEvent_t)h->ev_split, evp = early ? (cudaEvent_t)h->ev_plan : nullptr;
    const int sc = h->scatter_ctas > 0 ? h->scatter_ctas : h->num_sms;
    auto* dsc = (early && h->scatter_after_count) ? &run.scatter : nullptr;
    if (narrow)
      launch_hs<true>(src, q, recv, g, h->num_sms, L, mat, bstart, sst, ctl, fine, po, rec, idx,
                      &dplan->err, s, o.bmp, early, ls, evs, evp, sc, dsc);
    else
      launch_hs<false>(src, q, recv, g, h->num_sms, L, mat, bstart, sst, ctl, fine, po, rec, idx,
                       &dplan->err, s, o.bmp, early, ls, evs, evp, sc, dsc);
  }
  // the scatter set the occupancy bits: from here the local pass (on `ls`)
  // and the caller's stream (directory, lists) proceed independently
  const uint32_t* lfail = spec ? &dplan->spec_fail : po.fail;
  // CK holds the LSD composite (in-bucket key bits, combined index) of final
  // buckets wider than the box-count path; with HEADS every final bucket
  // spans <= 2^kLcSmallBits keys unless the refined sub-bins are wider, and
  // the box-count path ranks without composites, so 32-bit CK (less shared
  // memory: 3 resident CTAs per SM instead of 2) is enough
  const bool lsd_possible = !heads || final_span_bits(g) > kLcSmallBits;
  const bool ck32 = !lsd_possible || g.shift + g.cbits <= 32;
  // multi-GPU: the local pass writes local input indices; their global
  // indices follow in one high-occupancy gather (k_gid_map) instead of
  // latency-exposed lookups inside the local pass
  LocalOut ol = o;
  ol.gid[0] = ol.gid[1] = nullptr;
  ol.bmp[0] = ol.bmp[1] = nullptr;  // bits already set by the scatter
  const PlanOut pl = po;
  // beside the directory and the lists (late structure, or the partitioned
  // sort's deferred join) the local pass keeps two CTAs per SM so the other
  // stream's kernels find room (c4, 2^24 points: 2.15 vs 2.16 ms per step,
  // round 1 2.28 vs 2.43); from 2^25 points on its longer pass takes all
  // three (c2: 2.64 vs 2.655 ms)
  const int lcap = (!early && ls != s && g.n + g.m < (int64_t)1 << 25) ? 2 : 0;
  auto local = [=](cudaStream_t st) {
    if (spec_tail) spec_tail(st);
#define FMMB_LOCAL(CK, NW, HD)                                                                 \
  launch_local<CK, NW, HD>(h, rec, idx, pl.bstart_f, rbase, pl.desc, pl.nfinal, g, L, ol, lst, \
                           lfail, lcap, st)
    if (heads) {
      if (narrow) { if (ck32) FMMB_LOCAL(uint32_t, true, true); else FMMB_LOCAL(uint64_t, true, true); }
      else { if (ck32) FMMB_LOCAL(uint32_t, false, true); else FMMB_LOCAL(uint64_t, false, true); }
    } else {
      if (narrow) { if (ck32) FMMB_LOCAL(uint32_t, true, false); else FMMB_LOCAL(uint64_t, true, false); }
      else { if (ck32) FMMB_LOCAL(uint32_t, false, false); else FMMB_LOCAL(uint64_t, false, false); }
    }
#undef FMMB_LOCAL
    fmmb_trace_point(h, "local pass", st);
    if (q && n > 0 && o.q && !g.qrec)
      k_gather_q<<<(unsigned)h->num_sms * 16, 256, 0, st>>>(o.perm, q, n, o.q, lfail);
    if (o.gid[0] || o.gid[1])
      k_gid_map<<<(unsigned)h->num_sms * 16, 256, 0, st>>>(o.perm, n, m, o.gid[0], o.gid[1],
                                                            lfail);
    fmmb_trace_point(h, "charge gather", st);
  };
  // spec: init, scatter, counts, scan; hist: hist, scan, [fine], plan, scatter; + local
  const int sort_kernels = spec ? 4 : (g.shift > kLcSmallBits ? 4 : 5);
  launches += sort_kernels + 1 + ((o.gid[0] || o.gid[1]) ? 1 : 0) +
              ((q && n > 0 && o.q && !g.qrec) ? 1 : 0);
  run.local = local;
  run.scratch = w;
  run.g = g;
  run.bstart_f = po.bstart_f;
  run.rbase = rbase;
  run.desc = po.desc;
  run.nfinal = po.nfinal;
  run.hpos = idx;
  return FMMB_OK;
}

// ---- sort phase, general path: encode + Onesweep LSD + permuted gather
template <typename KeyT>
fmmb_status sort_onesweep(fmmb_handle_t h, const double* src, const double* q, int64_t n,
                          const double* recv, int64_t m, int L, const LocalOut& o,
                          BuildPlanHost* dplan, cudaStream_t s, int64_t& launches) {
  const int64_t tot = n + m;
  const int npass = sort_passes(L);
  const int64_t sort_tiles = ceil_div(tot, kSortTile);
  const int64_t gather_tiles = ceil_div(tot, kGTile);
  Carver c;
  const size_t o_hist = c.take<uint32_t>(npass * kBins);
  const size_t o_tc = c.take<uint32_t>(16);
  const size_t o_sst = c.take<uint64_t>((int64_t)npass * sort_tiles * kBins);
  const size_t o_gst = c.take<uint64_t>(gather_tiles);
  const size_t zero_bytes = c.off;
  const size_t o_ka = c.take<KeyT>(tot), o_kb = c.take<KeyT>(tot);
  const size_t o_va = c.take<uint32_t>(tot), o_vb = c.take<uint32_t>(tot);
  char* w = nullptr;
  if (cudaMallocAsync((void**)&w, c.off, s) != cudaSuccess)
    return fmmb_fail(h, FMMB_ERR_CUDA, "sort scratch of %zu bytes failed", c.off);
  cudaMemsetAsync(w, 0, zero_bytes, s);
  uint32_t* hist = (uint32_t*)(w + o_hist);
  uint32_t* tc = (uint32_t*)(w + o_tc);
  KeyT* ka = (KeyT*)(w + o_ka);
  KeyT* kb = (KeyT*)(w + o_kb);
  uint32_t* va = (uint32_t*)(w + o_va);
  uint32_t* vb = (uint32_t*)(w + o_vb);
  const int eg = (int)std::min<int64_t>(ceil_div(tot, kSortThreads), (int64_t)h->num_sms * 8);
  k_encode_hist<KeyT><<<eg, kSortThreads, 0, s>>>(src, n, recv, m, L, npass, ka, hist,
                                                  &dplan->err);
  ++launches;
  uint64_t* sst = (uint64_t*)(w + o_sst);
  const size_t smem = onesweep_smem_bytes(sizeof(KeyT));
  for (int ps = 0; ps < npass; ++ps) {
    uint64_t* st = sst + (size_t)ps * sort_tiles * kBins;
    if (ps == 0)
      k_onesweep<KeyT, true><<<(unsigned)sort_tiles, kSortThreads, smem, s>>>(
          ka, nullptr, kb, vb, tot, 0, hist, st, tc + ps);
    else
      k_onesweep<KeyT, false><<<(unsigned)sort_tiles, kSortThreads, smem, s>>>(
          ka, va, kb, vb, tot, kRadixBits * ps, hist + ps * kBins, st, tc + ps);
    ++launches;
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  k_gather<KeyT><<<(unsigned)gather_tiles, kGThreads, gather_smem_bytes(), s>>>(
      ka, va, n, m, L, src, q, recv, o.pts, o.q, o.perm, o.boxes, o.ne, o.bm, o.bmp[0], o.bmp[1],
      (uint64_t*)(w + o_gst), tc + 8, o.kinfo, o.gid[0], o.gid[1]);
  ++launches;
  cudaFreeAsync(w, s);
  return FMMB_OK;
}

// E2/E4 write pass (warp per receiver parent, grid-stride).  `sparse`: the
// finest level's rows average well under the 189 entries of a full window
// (surfaces, clustered inputs) -- the member-compacting variant visits only
// the chunks holding occupied members (c3: 0.56 vs 0.64 ms; the dense
// variant keeps c2 at 1.09 ms)
inline void launch_lists_write(fmmb_handle_t h, const ListsParams& lp, const ListsLayout* lay,
                               int64_t nwork_cap, bool sparse, cudaStream_t s) {
  const int lgrid = (int)std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(nwork_cap, kLWarps), (int64_t)h->num_sms * h->lw_per_sm));
  if (sparse) k_lists_write<true><<<lgrid, kLThreads, 0, s>>>(lp, lay);
  else k_lists_write<false><<<lgrid, kLThreads, 0, s>>>(lp, lay);
}
inline bool lists_sparse(int64_t e4_rows_entries, int64_t rows) {
  return rows > 0 && e4_rows_entries < 120 * rows;
}

// Multi-GPU sort phase extras: global indices of the local points and the
// caller's level-L occupancy bitmaps (src words then recv words).
struct DistSortArgs {
  const int64_t* gid_src;
  const int64_t* gid_recv;
  uint64_t* bmp;
  bool defer_join;  // leave the local pass running on the side stream (fmmb_dist_join)
};

template <typename KeyT>
fmmb_status build_impl(fmmb_handle_t h, const double* src, const double* q, int64_t n,
                       const double* recv, int64_t m, int L, fmmb_alloc_fn alloc,
                       void* ctx, fmmb_structures* out, cudaEvent_t* ev,
                       cudaStream_t s, bool lists, const DistSortArgs* dsa = nullptr) {
  const int64_t tot = n + m;
  const int stride = L + 1;
  // level-L occupancy bitmaps + rank directory drive the bucket path's heads
  // pass: always with lists, and for the partitioned sort (dsa->bmp wanted)
  const bool heads = lists || (dsa && dsa->bmp);

  // bitmap segment layout: seg = set*(L+1)+l, each starting on a rank tile
  RankParams rp{};
  rp.nseg = 2 * stride;
  int64_t words = 0, tiles = 0;
  for (int set = 0; set < 2; ++set)
    for (int l = 0; l <= L; ++l) {
      const int sg = set * stride + l;
      rp.word_off[sg] = words;
      rp.nwords[sg] = level_words(l);
      rp.tile_off[sg] = tiles;
      const int64_t t = ceil_div(rp.nwords[sg], kRTileWords);
      tiles += t;
      words += t * kRTileWords;
    }
  rp.tile_off[rp.nseg] = tiles;
  const int64_t bmp_words = heads ? words : 0, rank_tiles = heads ? tiles : 0;

  // count-scan tiles: capacity from min(m, 8^(l-1)) receiver parents per level
  int64_t cs_tiles = 1;
  for (int l = std::max(1, lists_lmin_host(L)); l <= L; ++l)
    cs_tiles += ceil_div(cap_level(m, l - 1), kCsParents);
  // ---- workspace: [zeroed control | rest]
  Carver z;
  const size_t o_tc = z.take<uint32_t>(16);  // tile counters
  const size_t o_rst = z.take<uint64_t>(rank_tiles);
  const size_t o_st4 = z.take<uint64_t>(lists ? cs_tiles : 0);
  const size_t o_st2 = z.take<uint64_t>(lists ? cs_tiles : 0);
  const size_t o_plan = z.take<BuildPlanHost>(1);
  const size_t o_bmp = z.take<uint64_t>(bmp_words);
  const size_t zero_bytes = z.off;
  const size_t o_dir = z.take<uint32_t>(bmp_words);
  const size_t o_lowkeys = z.take<uint64_t>(2 * (1 + 8));  // levels 0,1 keys
  const size_t o_lay = z.take<ListsLayout>(1);

  char* ws = nullptr;
  if (cudaMallocAsync((void**)&ws, z.off, s) != cudaSuccess)
    return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation of %zu bytes failed", z.off);
  auto W = [&](size_t o) { return (void*)(ws + o); };
  uint32_t* tc = (uint32_t*)W(o_tc);
  BuildPlanHost* dplan = (BuildPlanHost*)W(o_plan);
  uint64_t* bmp = (uint64_t*)W(o_bmp);
  uint32_t* dir = (uint32_t*)W(o_dir);

  // ---- output arena A (sizes known before the build)
  Carver a;
  const size_t a_pts = a.take<double>(3 * tot);
  const size_t a_q = a.take<double>(q ? n : 0);
  const size_t a_perm = a.take<int64_t>(tot);
  const size_t a_boxes = a.take<uint64_t>(tot);
  const size_t a_ne = a.take<uint64_t>(tot);
  const size_t a_bm = a.take<int64_t>(tot + 2);
  size_t a_dir[2][kMaxLevel + 1] = {};
  size_t a_lbm[kMaxLevel + 1] = {};
  if (lists) {
    for (int l = 2; l < L; ++l) {
      a_dir[0][l] = a.take<uint64_t>(cap_level(n, l));
      a_dir[1][l] = a.take<uint64_t>(cap_level(m, l));
    }
    a_lbm[0] = a.take<int64_t>(cap_level(m, L) + 1);
    for (int l = 2; l <= L; ++l) a_lbm[l] = a.take<int64_t>(cap_level(m, l) + 1);
  }
  char* arena = (char*)alloc(ctx, a.off);
  if (!arena) {
    cudaFreeAsync(ws, s);
    return fmmb_fail(h, FMMB_ERR_ALLOC, "output allocation of %zu bytes failed", a.off);
  }
  auto A = [&](size_t o) { return (void*)(arena + o); };
  double* pts_out = (double*)A(a_pts);
  int64_t* bm_out = (int64_t*)A(a_bm);
  uint64_t* ne_out = (uint64_t*)A(a_ne);

  LocalOut lo{};
  lo.pts = pts_out;
  lo.q = q ? (double*)A(a_q) : nullptr;
  lo.perm = (int64_t*)A(a_perm);
  lo.boxes = (uint64_t*)A(a_boxes);
  lo.ne = ne_out;
  lo.bm = bm_out;
  lo.bmp[0] = heads ? (unsigned long long*)(bmp + rp.word_off[L]) : nullptr;
  lo.bmp[1] = heads ? (unsigned long long*)(bmp + rp.word_off[stride + L]) : nullptr;
  lo.kinfo = dplan->kinfo;
  if (dsa) {
    lo.gid[0] = dsa->gid_src;
    lo.gid[1] = dsa->gid_recv;
  }

  int64_t launches = 0;
  bool fast = h->sort_path != 2 && tot > 0 && bucket_fits(bucket_geo(L, n, m, h->num_sms));
  // speculative bucket regions (no histogram pass) unless this shape missed last time
  bool spec = fast && h->sort_path != 3 && spec_possible(bucket_geo(L, n, m, h->num_sms)) &&
              !(h->spec_miss_level == L && h->spec_miss_n == n && h->spec_miss_m == m);
  BuildPlanHost* hp = (BuildPlanHost*)h->pinned;
  ListsParams lp{};
  int64_t nwork_cap = 0;
  // local pass + heads stream (== s unless the bucket path overlaps them
  // with the directory / lists); join() orders s after its work
  cudaStream_t ls = s;
  auto join = [&]() {
    if (ls != s) cudaStreamWaitEvent(s, (cudaEvent_t)h->ev_side, 0);
  };
  // Dense geometries (>= 4 points per finest box on average: every row is
  // full, so the per-row bounds E4 <= 189, E2 <= 27 overshoot the real list
  // sizes by a few percent): the list arena is allocated up front at those
  // bounds and the write pass is enqueued right behind the count -- the host
  // waits for the size read-back only, not before launching the write.
  const bool upfront = lists && L >= 2 && h->lists_upfront &&
                       (double)m >= 4.0 * std::ldexp(1.0, 3 * L);
  if (upfront) {
    Carver b;
    const size_t b_e2 = b.take<int64_t>(27 * cap_level(m, L));
    size_t b_r[kMaxLevel + 1] = {}, b_c[kMaxLevel + 1] = {};
    for (int k = 2; k <= L; ++k) {
      b_r[k] = b.take<int64_t>(189 * cap_level(m, k));
      b_c[k] = b.take<int16_t>(189 * cap_level(m, k));
    }
    char* arena_b = (char*)alloc(ctx, std::max<size_t>(b.off, 256));
    if (!arena_b) {
      cudaFreeAsync(ws, s);
      return fmmb_fail(h, FMMB_ERR_ALLOC, "list allocation of %zu bytes failed", b.off);
    }
    lp.ranks_out[0] = (int64_t*)(arena_b + b_e2);
    for (int k = 2; k <= L; ++k) {
      lp.ranks_out[k] = (int64_t*)(arena_b + b_r[k]);
      lp.codes_out[k] = (int16_t*)(arena_b + b_c[k]);
    }
  }
  for (int attempt = 0;; ++attempt) {
    h->tr_n = 0;
    fmmb_trace_point(h, "start", s);
    if (ev) cudaEventRecord(ev[0], s);
    cudaMemsetAsync(ws, 0, zero_bytes, s);
    if (tot == 0) cudaMemsetAsync(bm_out, 0, 2 * sizeof(int64_t), s);

    // ---- K1-K4: sort both sets into the reference layout
    BucketRun brun;
    ls = (fast && heads && h->overlap && h->side) ? (cudaStream_t)h->side : s;
    // early occupancy: the histogram pass sets the level-L bits and the sort
    // continues on the side stream while this stream builds the directory
    // and the lists (which need nothing but the bitmaps)
    // (chosen when the histogram pass runs anyway -- wide or skewed
    // geometries, c3: measured 3.57 vs 3.71 ms; with speculative regions
    // the scatter sets the bits itself -- c2: 3.04 vs 3.19 ms)
    const bool early = fast && lists && !dsa && ls != s &&
                       (h->early_occ == 2 || (h->early_occ == 1 && !spec));
    if (early) {
      spec = false;
      ls = (cudaStream_t)h->side_hi;  // the sort chain is the critical path
    }
    if (tot > 0) {
      const fmmb_status st =
          fast ? sort_bucket(h, src, q, n, recv, m, L, lo, heads, spec, dplan, s, launches, brun,
                             ls, early)
               : sort_onesweep<KeyT>(h, src, q, n, recv, m, L, lo, dplan, s, launches);
      if (st != FMMB_OK) {
        join();
        cudaFreeAsync(ws, s);
        return st;
      }
    }
    // the local pass on the side stream: right after the scatter (it then
    // overlaps the directory, the count and the write), or after the count
    // when h->local_after_count (A/B knob FMMB_LOCAL_AFTER=1)
    auto start_local = [&]() {
      if (!brun.local) return;
      if (ls != s && !early) {  // (early: the scatter already runs on ls)
        cudaEventRecord((cudaEvent_t)h->ev_split, s);
        cudaStreamWaitEvent(ls, (cudaEvent_t)h->ev_split, 0);
      }
      brun.local(ls);
      brun.local = nullptr;
    };
    fmmb_trace_point(h, early ? "hist+occupancy (s)" : "sort (s)", s);
    if (early && !brun.scatter) fmmb_trace_point(h, "scan+plan+scatter (side)", ls);
    if ((!h->local_after_count || !lists) && !brun.scatter) start_local();
    if (ev) cudaEventRecord(ev[1], s);

    // ---- K5: bitmap pyramid (big levels one launch each, the rest in one CTA)
    int l = lists ? L : 0;
    while (l >= 1 && level_words(l - 1) > 256) {
      const int64_t nc = level_words(l - 1);
      k_pyramid<<<(unsigned)ceil_div(2 * nc, 256), 256, 0, s>>>(
          bmp + rp.word_off[l], bmp + rp.word_off[l - 1], bmp + rp.word_off[stride + l],
          bmp + rp.word_off[stride + l - 1], nc);
      ++launches;
      --l;
    }
    if (l >= 1) {
      PyramidTail pt{};
      for (int k = 0; k <= L; ++k) {
        pt.lvl[0][k] = bmp + rp.word_off[k];
        pt.lvl[1][k] = bmp + rp.word_off[stride + k];
        pt.nwords[k] = level_words(k);
      }
      pt.from_level = l;
      k_pyramid_tail<<<1, 1024, 0, s>>>(pt);
      ++launches;
    }
    // ---- rank directory, totals and per-level directory keys
    rp.bmp = bmp;
    rp.dir = dir;
    rp.states = (uint64_t*)W(o_rst);
    rp.tile_counter = tc + 9;
    rp.totals = dplan->ktot;
    uint64_t* lowkeys = (uint64_t*)W(o_lowkeys);
    for (int set = 0; set < 2; ++set)
      for (int k = 0; k <= L; ++k) {
        uint64_t* dst = nullptr;
        if (k < L) {
          if (k == 0) dst = lowkeys + set * 9;
          else if (k == 1) dst = lowkeys + set * 9 + 1;
          else if (lists) dst = (uint64_t*)A(a_dir[set][k]);
        }
        rp.keys_out[set * stride + k] = dst;
      }
    if (heads) {
      k_rank<<<(unsigned)rank_tiles, kRThreads, 0, s>>>(rp);
      ++launches;
    }
    fmmb_trace_point(h, "pyramid+rank (s)", s);
    if (dsa && dsa->bmp) {  // this rank's level-L occupancy, for the all-reduce
      cudaMemcpyAsync(dsa->bmp, bmp + rp.word_off[L], level_words(L) * sizeof(uint64_t),
                      cudaMemcpyDeviceToDevice, s);
      cudaMemcpyAsync(dsa->bmp + level_words(L), bmp + rp.word_off[stride + L],
                      level_words(L) * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s);
    }
    if (ev) cudaEventRecord(ev[2], s);

    nwork_cap = 0;
    if (lists) {
      lp.level = L;
      lp.dense_rows = h->dense_rows;
      lp.key_lo = 0;
      lp.key_hi = 1ull << (3 * L);
      lp.ktot = dplan->ktot;
      lp.bmp = bmp;
      lp.dir = dir;
      for (int set = 0; set < 2; ++set)
        for (int k = 0; k <= L; ++k) lp.bmp_off[set][k] = rp.word_off[set * stride + k];
      for (int k = 0; k < L; ++k) lp.rkeys[k] = rp.keys_out[stride + k];
      lp.bm[0] = (int64_t*)A(a_lbm[0]);
      for (int k = 2; k <= L; ++k) lp.bm[k] = (int64_t*)A(a_lbm[k]);
      for (int k = std::max(1, lists_lmin_host(L)); k <= L; ++k) nwork_cap += cap_level(m, k - 1);
      if (L == 0) nwork_cap = 1;
      const int lgrid = (int)std::max<int64_t>(
          1, std::min<int64_t>(ceil_div(nwork_cap, kLWarps), (int64_t)h->num_sms * 16));
      ListsLayout* glay = (ListsLayout*)W(o_lay);
      k_lists_plan<<<1, 32, 0, s>>>(lp, glay);
      // a loose tile bound (deep, sparse levels) gets a persistent grid
      const bool cs_loop = h->cs_per_sm > 0 || cs_tiles > (int64_t)h->num_sms * 32;
      if (cs_loop)
        k_lists_cscan<true><<<(unsigned)(h->num_sms * (h->cs_per_sm > 0 ? h->cs_per_sm : 8)),
                              kLThreads, 0, s>>>(
            lp, glay, (uint64_t*)W(o_st4), (uint64_t*)W(o_st2), tc + 10, dplan->seg_totals);
      else
        k_lists_cscan<false><<<(unsigned)cs_tiles, kLThreads, 0, s>>>(
            lp, glay, (uint64_t*)W(o_st4), (uint64_t*)W(o_st2), tc + 10, dplan->seg_totals);
      launches += 2;
      fmmb_trace_point(h, "lists count (s)", s);
    }
    if (brun.scatter) {  // early occupancy: the scatter starts once the count has its SMs
      cudaEventRecord((cudaEvent_t)h->ev_count, s);
      cudaStreamWaitEvent(ls, (cudaEvent_t)h->ev_count, 0);
      brun.scatter(ls);
      brun.scatter = nullptr;
      fmmb_trace_point(h, "scatter (side)", ls);
    }
    start_local();
    if (brun.scratch) {  // bucket path: bookmarks / non-empty keys at global box ranks
      if (ls != s) {  // heads on the side stream: after the local pass and the rank directory
        cudaEventRecord((cudaEvent_t)h->ev_rank, s);
        cudaStreamWaitEvent(ls, (cudaEvent_t)h->ev_rank, 0);
      }
      if (heads) {
        HeadsParams hpar{};
        for (int set = 0; set < 2; ++set) {
          hpar.bmp[set] = bmp + rp.word_off[set * stride + L];
          hpar.dir[set] = dir + rp.word_off[set * stride + L];
        }
        hpar.ktot_src = dplan->ktot + L;
        hpar.ktot_recv = dplan->ktot + stride + L;
        hpar.bstart = brun.bstart_f;
        hpar.rbase = brun.rbase;
        hpar.hpos = brun.hpos;
        hpar.ne = ne_out;
        hpar.bm = bm_out;
        hpar.kinfo = dplan->kinfo;
        k_bkt_heads<<<(unsigned)h->num_sms * 8, 256, 0, ls>>>(hpar, brun.desc, brun.nfinal,
                                                               brun.g);
        ++launches;
        fmmb_trace_point(h, ls != s ? "heads (side)" : "heads (s)", ls);
      }
      cudaFreeAsync(brun.scratch, ls);
    }
    if (ls != s) cudaEventRecord((cudaEvent_t)h->ev_side, ls);
    if (ev) cudaEventRecord(ev[3], s);

    // ---- sizes back to the host (the build's single synchronisation); early
    // occupancy: the sort stream's refinement plan (overflow flag) first
    if (early && tot > 0) cudaStreamWaitEvent(s, (cudaEvent_t)h->ev_plan, 0);
    cudaMemcpyAsync(hp, dplan, sizeof(BuildPlanHost), cudaMemcpyDeviceToHost, s);
    cudaEventRecord((cudaEvent_t)h->ev_rb, s);
    fmmb_trace_point(h, "size read-back (s)", s);
    if (upfront) {  // the write right behind the count (sizes are not needed for it)
      if (ev) cudaEventRecord(ev[4], s);
      launch_lists_write(h, lp, (const ListsLayout*)W(o_lay), nwork_cap, false, s);
      ++launches;
      fmmb_trace_point(h, "lists write (s)", s);
      if (ev) cudaEventRecord(ev[5], s);
    }
    cudaError_t ce = cudaEventSynchronize((cudaEvent_t)h->ev_rb);
    if (ce != cudaSuccess) {
      join();
      cudaFreeAsync(ws, s);
      return fmmb_fail(h, FMMB_ERR_CUDA, "build phase A failed: %s", cudaGetErrorString(ce));
    }
    if (spec && hp->spec_fail && attempt < 2) {  // a speculative region overflowed
      join();
      h->spec_miss_level = L;
      h->spec_miss_n = n;
      h->spec_miss_m = m;
      spec = false;
      continue;
    }
    if (hp->fail && fast && attempt < 2) {  // a bucket overflowed: general sort
      join();
      fast = false;
      spec = false;
      continue;
    }
    break;
  }
  if (hp->fail) {
    join();
    cudaFreeAsync(ws, s);
    return fmmb_fail(h, FMMB_ERR_CUDA, "internal: bucket sort overflow after fallback");
  }
  h->last_sort_path = fast ? 1 : 2;
  if (hp->err) {
    join();
    cudaFreeAsync(ws, s);
    return fmmb_fail(h, FMMB_ERR_DOMAIN,
                     "a point's Morton index lies outside the level-%d grid "
                     "(coordinates must lie in the unit cube)", L);
  }
  const int64_t ks = heads ? hp->ktot[L] : (n > 0 ? hp->kinfo[0] : 0);
  const int64_t kr = heads ? hp->ktot[stride + L] : (m > 0 ? hp->kinfo[1] - ks : 0);
  // (kinfo comes from the heads pass; overlapped, it is not read back yet)
  if (heads && ls == s && tot > 0 &&
      (hp->kinfo[0] != ks || (m > 0 && hp->kinfo[1] != ks + kr))) {
    join();
    cudaFreeAsync(ws, s);
    return fmmb_fail(h, FMMB_ERR_CUDA, "internal: box counts disagree (%lld/%lld vs %lld/%lld)",
                     (long long)hp->kinfo[0], (long long)hp->kinfo[1], (long long)ks,
                     (long long)kr);
  }

  // ---- fill the output descriptor (phase A part)
  memset(out, 0, sizeof(*out));
  out->max_level = L;
  out->src.points = pts_out;
  out->src.charges = q ? (double*)A(a_q) : nullptr;
  out->src.permutation = (int64_t*)A(a_perm);
  out->src.boxes = (uint64_t*)A(a_boxes);
  out->src.non_empty = ne_out;
  out->src.bookmarks = bm_out;
  out->src.n = n;
  out->src.k = ks;
  out->recv.points = pts_out + 3 * n;
  out->recv.charges = nullptr;
  out->recv.permutation = (int64_t*)A(a_perm) + n;
  out->recv.boxes = (uint64_t*)A(a_boxes) + n;
  out->recv.non_empty = ne_out + ks;
  out->recv.bookmarks = bm_out + ks + 1;
  out->recv.n = m;
  out->recv.k = kr;

  if (lists) {
    // ---- phase B: exactly-sized list outputs, then the write pass
    const int64_t e2 = hp->seg_totals[0];
    if (!upfront) {
    Carver b;
    const size_t b_e2 = b.take<int64_t>(e2);
    size_t b_r[kMaxLevel + 1] = {}, b_c[kMaxLevel + 1] = {};
    for (int k = 2; k <= L; ++k) {
      b_r[k] = b.take<int64_t>(hp->seg_totals[k]);
      b_c[k] = b.take<int16_t>(hp->seg_totals[k]);
    }
    char* arena_b = (char*)alloc(ctx, std::max<size_t>(b.off, 256));
    if (!arena_b) {
      join();
      cudaFreeAsync(ws, s);
      return fmmb_fail(h, FMMB_ERR_ALLOC, "list allocation of %zu bytes failed", b.off);
    }
    lp.ranks_out[0] = (int64_t*)(arena_b + b_e2);
    for (int k = 2; k <= L; ++k) {
      lp.ranks_out[k] = (int64_t*)(arena_b + b_r[k]);
      lp.codes_out[k] = (int16_t*)(arena_b + b_c[k]);
    }
    if (ev) cudaEventRecord(ev[4], s);
    fmmb_trace_point(h, "host: list arena (s)", s);
    launch_lists_write(h, lp, (const ListsLayout*)W(o_lay), nwork_cap,
                       lists_sparse(L >= 2 ? hp->seg_totals[L] : 0, kr), s);
    ++launches;
    fmmb_trace_point(h, "lists write (s)", s);
    if (ev) cudaEventRecord(ev[5], s);  // the write kernel alone (before the side join)
    }

    out->neighbor_bookmark = lp.bm[0];
    out->neighbor_list = lp.ranks_out[0];
    out->n_neighbor = e2;
    out->dir_src[L] = ne_out;
    out->n_dir_src[L] = ks;
    out->dir_recv[L] = ne_out + ks;
    out->n_dir_recv[L] = kr;
    for (int k = 2; k < L; ++k) {
      out->dir_src[k] = (uint64_t*)A(a_dir[0][k]);
      out->dir_recv[k] = (uint64_t*)A(a_dir[1][k]);
      out->n_dir_src[k] = hp->ktot[k];
      out->n_dir_recv[k] = hp->ktot[stride + k];
    }
    for (int k = 2; k <= L; ++k) {
      out->st_bookmark[k] = lp.bm[k];
      out->st_ranks[k] = lp.ranks_out[k];
      out->st_codes[k] = lp.codes_out[k];
      out->n_st[k] = hp->seg_totals[k];
    }
  }
  // the caller's stream sees the local pass and heads complete (the
  // partitioned sort defers this: its bitmap all-reduce and owned lists only
  // need the occupancy, fmmb_dist_join orders the caller after the rest)
  const bool deferred = dsa && dsa->defer_join && ls != s;
  if (!deferred) join();
  fmmb_trace_point(h, "joined (s)", s);
  if (ev) {
    if (!lists) {
      cudaEventRecord(ev[4], s);
      cudaEventRecord(ev[5], s);
    }
  }
  // (deferred: the heads pass on the side stream still reads the directory)
  cudaFreeAsync(ws, deferred ? ls : s);
  out->n_launches = launches;
  h->launches = launches;
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess)
    return fmmb_fail(h, FMMB_ERR_CUDA, "build launch failed: %s", cudaGetErrorString(ce));
  return FMMB_OK;
}

fmmb_status check_build_args(fmmb_handle_t h, const double* src, int64_t n, const double* recv,
                             int64_t m, int level, fmmb_alloc_fn alloc, bool lists) {
  if (!h) return FMMB_ERR_ARG;
  if (level < 0 || level > kMaxLevel)
    return fmmb_fail(h, FMMB_ERR_CAPACITY, "max_level %d outside [0, %d]", level, kMaxLevel);
  if (n < 0 || m < 0 || (n > 0 && !src) || (m > 0 && !recv) || !alloc)
    return fmmb_fail(h, FMMB_ERR_ARG, "invalid arguments");
  if (n + m >= (1ll << 31))
    return fmmb_fail(h, FMMB_ERR_CAPACITY, "n + m = %lld exceeds 2^31 - 1 points per device",
                     (long long)(n + m));
  if (lists && !fmmb_bitmap_ok(level, n + m))
    return fmmb_fail(h, FMMB_ERR_CAPACITY,
                     "level %d occupancy bitmaps exceed the device budget for %lld points",
                     level, (long long)(n + m));
  return FMMB_OK;
}

}  // namespace


extern "C" fmmb_status fmmb_build_all(fmmb_handle_t h, const double* src, const double* charges,
                                      int64_t n, const double* recv, int64_t m, int level,
                                      fmmb_alloc_fn alloc, void* ctx, fmmb_structures* out,
                                      void** timing, void* stream) {
  FMMB_GUARD(h);
  fmmb_status st = check_build_args(h, src, n, recv, m, level, alloc, true);
  if (st != FMMB_OK) return st;
  if (!out) return FMMB_ERR_ARG;
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)timing;
  if (sort_key_bits(level) <= 32)
    return build_impl<uint32_t>(h, src, charges, n, recv, m, level, alloc, ctx, out, ev, s, true);
  return build_impl<uint64_t>(h, src, charges, n, recv, m, level, alloc, ctx, out, ev, s, true);
}

extern "C" fmmb_status fmmb_sort_points(fmmb_handle_t h, const double* points,
                                        const double* charges, int64_t n, int level,
                                        fmmb_alloc_fn alloc, void* ctx, fmmb_point_set* out,
                                        void* stream) {
  FMMB_GUARD(h);
  fmmb_status st = check_build_args(h, points, n, nullptr, 0, level, alloc, false);
  if (st != FMMB_OK) return st;
  if (!out) return FMMB_ERR_ARG;
  cudaSetDevice(h->device);
  fmmb_structures tmp;
  cudaStream_t s = (cudaStream_t)stream;
  if (sort_key_bits(level) <= 32)
    st = build_impl<uint32_t>(h, points, charges, n, nullptr, 0, level, alloc, ctx, &tmp,
                              nullptr, s, false);
  else
    st = build_impl<uint64_t>(h, points, charges, n, nullptr, 0, level, alloc, ctx, &tmp,
                              nullptr, s, false);
  if (st == FMMB_OK) *out = tmp.src;
  return st;
}

#include "plugin.cuh"
#include "dist_api.cuh"
#include "nearfield.cuh"
#include "boxtype.cuh"
#include "partplan.cuh"
#include "workload.cuh"
