// Host-side internals shared by the libfmmb200 translation units.
#pragma once
#include <stdint.h>

#include <mutex>
#include <string>

#include "../../include/fmmb200.h"

struct fmmb_handle_s {
  int device = 0;
  int num_sms = 148;
  void* pinned = nullptr;  // small pinned block for size read-back
  int64_t launches = 0;
  int sort_path = 0;       // 0 auto (bucket sort, Onesweep on overflow), 1 bucket, 2 Onesweep
  int last_sort_path = 0;  // path the last build's sort phase completed on
  // geometry (level, n, m) whose speculative bucket regions last overflowed:
  // the next build of the same shape starts with the histogram pass
  int64_t spec_miss_level = -1, spec_miss_n = -1, spec_miss_m = -1;
  // side stream of the bucket path: the local pass + heads run there while
  // the caller's stream builds the directory and the lists (both only need
  // the occupancy bitmaps, which the scatter sets)
  void* side = nullptr;          // cudaStream_t
  void* side_hi = nullptr;       // cudaStream_t, highest priority (early-occupancy sort chain)
  void* ev_split = nullptr;      // cudaEvent_t: scatter done (caller stream)
  void* ev_rank = nullptr;       // rank directory done (caller stream)
  void* ev_side = nullptr;       // side stream's work done
  void* ev_plan = nullptr;       // early occupancy: refinement plan done (sort stream)
  void* ev_count = nullptr;      // early occupancy: list count done (caller stream)
  void* ev_rb = nullptr;         // size read-back done (the host waits on it)
  bool lists_upfront = true;     // dense geometries: list arena at the row bounds, write
                                 // enqueued before the host wait (FMMB_LISTS_EXACT=1: off)
  bool scatter_after_count = false;  // early occupancy: scatter waits for the list count
                                    // (FMMB_SCATTER_AFTER_COUNT=1; default: right after the plan)
  int early_occ = 1;             // occupancy bits from the histogram pass, sort on the side
                                 // stream beside the directory + lists: 1 when the histogram
                                 // pass runs anyway, 2 always (FMMB_EARLY_OCC=1), 0 never
                                 // (FMMB_LATE_OCC=1)
  bool rec_q = true;             // source records carry q + idx side store (FMMB_REC_IDX=1:
                                 // records carry the index, charges gathered after the sort)
  bool rec_embed = true;         // source index in the record's exponents where possible
  int scatter_ctas = 0;          // FMMB_SCATTER_CTAS: cap on the scatter's persistent grid (A/B)
  bool overlap = true;           // FMMB_NO_OVERLAP=1 serialises (A/B)
  bool local_after_count = false;  // FMMB_LOCAL_AFTER=1: local pass after the list count (A/B)
  int lc_per_sm = 0;   // FMMB_LC_PER_SM: cap on resident local-pass CTAs per SM (A/B)
  int dense_rows = 0;  // FMMB_DENSE_ROWS: row-by-row dense list writer (A/B)
  int lw_per_sm = 32;  // FMMB_LW_PER_SM: list-write grid in CTAs per SM (A/B)
  int cs_per_sm = 0;   // FMMB_CS_PER_SM: force the persistent list count at this many CTAs per SM
  // FMMB_TRACE=1: timing events at the phase boundaries of both streams of
  // the last build (fmmb_trace): the overlap timeline without a profiler
  bool trace = false;
  int tr_n = 0;
  void* tr_ev[32] = {};
  const char* tr_name[32] = {};
  // every entry point holds this for its whole call: the pinned read-back
  // block, the side stream and its events are per handle, so concurrent
  // callers on one device (the reference's kernels are nogil and reentrant,
  // SURVEY 8(b) "Threading") are serialised instead of racing on them
  std::recursive_mutex mu;
};

// null check + the handle's call lock for the rest of the entry point
#define FMMB_GUARD(h)                 \
  if (!(h)) return FMMB_ERR_ARG;      \
  std::lock_guard<std::recursive_mutex> fmmb_guard_((h)->mu)

constexpr size_t kPinnedBytes = 1 << 16;

fmmb_status fmmb_fail(fmmb_handle_t h, fmmb_status st, const char* fmt, ...);
bool fmmb_bitmap_ok(int level, int64_t n_total);
int lists_lmin_host(int L);
void fmmb_trace_point(fmmb_handle_t h, const char* name, void* stream);
