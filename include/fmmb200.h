/*
 * fmmb200.h — C ABI of libfmmb200.so, the B200-native (sm_100a) build of the
 * FMM data structures of Hu, Gumerov & Duraiswami (arXiv 1301.1704, Alg. 1-5).
 *
 * This is the drop-in boundary for the reference package `fmmkit`:
 *
 *   - the kernel plugin bound to `fmmkit.backend.kernels`
 *     (reference: pkg/src/fmmkit/backend.py:19-27, signatures in
 *      pkg/src/fmmkit/_ckernels.pyx:65-287 and _pykernels.py:22-197), and
 *   - the build API `fmmkit.build_all` / `fmmkit.sort_points`
 *     (reference: pkg/src/fmmkit/lists.py:133-187, pseudosort.py:138-151).
 *
 * Every entry point takes plain device pointers and element counts, is
 * stream-ordered on the caller's `stream` (a cudaStream_t passed as void*),
 * and returns an fmmb_status.  No torch / numpy types cross this boundary.
 * Outputs whose size is only known on the device are allocated through the
 * caller's allocator callback (so e.g. the PyTorch caching allocator owns
 * them); the library's temporary workspace is stream-ordered
 * (cudaMallocAsync) and released before the call returns.
 *
 * Error codes mirror the reference exception types (errors.py:4-21):
 *   FMMB_ERR_DOMAIN   -> fmmkit.errors.DomainError   (precondition violated)
 *   FMMB_ERR_CAPACITY -> fmmkit.errors.CapacityError (level cap / budget)
 * fmmb_last_error() returns the message of the calling thread's last failing
 * call (thread-local text).
 *
 * Threading: entry points are reentrant, like the reference's nogil kernels
 * (SURVEY 8(b)).  Each call holds its handle's lock for its duration (the
 * handle's pinned read-back block, side stream and events are per handle),
 * so concurrent calls on one handle from several host threads serialise and
 * each returns exactly what it would return alone; calls on different
 * streams are allowed (every workspace is per call).
 */
#ifndef FMMB200_H
#define FMMB200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FMMB_API __attribute__((visibility("default")))
#else
#define FMMB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define FMMB_MAX_LEVEL 20 /* morton.py:18 MAX_LEVEL */
#define FMMB_ABI_VERSION 1

typedef enum fmmb_status {
  FMMB_OK = 0,
  FMMB_ERR_DOMAIN = 1,   /* DomainError  (errors.py:12) */
  FMMB_ERR_CAPACITY = 2, /* CapacityError (errors.py:8)  */
  FMMB_ERR_CUDA = 3,     /* CUDA runtime failure          */
  FMMB_ERR_ALLOC = 4,    /* allocator callback returned NULL */
  FMMB_ERR_ARG = 5       /* NULL handle / pointer misuse  */
} fmmb_status;

typedef struct fmmb_handle_s* fmmb_handle_t;

/* Allocator callback: returns a device pointer of >= nbytes, aligned to 256 B,
 * valid on the call's stream; NULL on failure.  Called only from the host
 * thread that made the library call. */
typedef void* (*fmmb_alloc_fn)(void* ctx, uint64_t nbytes);

/* ---------------------------------------------------------------- lifecycle */
FMMB_API int fmmb_abi_version(void);
FMMB_API fmmb_status fmmb_create(int device, fmmb_handle_t* out);
FMMB_API fmmb_status fmmb_destroy(fmmb_handle_t h);
FMMB_API const char* fmmb_last_error(fmmb_handle_t h);
/* number of kernel launches issued by the last call on this handle */
FMMB_API int64_t fmmb_last_launch_count(fmmb_handle_t h);
/* Sort-phase strategy of fmmb_build_all / fmmb_sort_points (no reference
 * counterpart; both strategies give bit-identical outputs):
 *   0 = auto: payload-carrying bucket sort, rerun on the Onesweep path if a
 *       bucket overflows the bucket sort's shared-memory capacity;
 *   1 = bucket sort (with the same overflow rerun);  2 = Onesweep LSD + gather;
 *   3 = bucket sort without speculative fixed regions (histogram pass first).
 * fmmb_last_sort_path() reports the path the last build completed on (1/2). */
FMMB_API fmmb_status fmmb_set_sort_path(fmmb_handle_t h, int path);
FMMB_API int fmmb_last_sort_path(fmmb_handle_t h);
/* Phase timeline of the last fmmb_build_all when the handle was created with
 * FMMB_TRACE=1 in the environment (0 entries otherwise): ms[i] since the
 * build's start event and a static phase name, for up to `cap` boundaries,
 * recorded on the stream that ran the phase (caller's or side stream). */
FMMB_API int fmmb_trace(fmmb_handle_t h, float* ms, const char** names, int cap);
/* Bucket path stream structure: 1 (default) = the local pass and the heads
 * pass run on an internal side stream, concurrently with the directory and
 * the lists on the caller's stream (joined before the call returns);
 * 0 = everything in order on the caller's stream.  Outputs are identical. */
FMMB_API fmmb_status fmmb_set_overlap(fmmb_handle_t h, int on);

/* ------------------------------------------------------ kernel plugin level */

/* spread_bits / compact_bits  (_pykernels.py:22-40, _ckernels.pyx:27-44,65-70) */
FMMB_API fmmb_status fmmb_spread_bits(fmmb_handle_t h, const uint64_t* v, int64_t n,
                             uint64_t* out, void* stream);
FMMB_API fmmb_status fmmb_compact_bits(fmmb_handle_t h, const uint64_t* v, int64_t n,
                              uint64_t* out, void* stream);
/* interleave_coords / deinterleave_indices (_pykernels.py:43-57) */
FMMB_API fmmb_status fmmb_interleave_coords(fmmb_handle_t h, const uint64_t* ix,
                                   const uint64_t* iy, const uint64_t* iz,
                                   int64_t n, uint64_t* out, void* stream);
FMMB_API fmmb_status fmmb_deinterleave_indices(fmmb_handle_t h, const uint64_t* idx,
                                      int64_t n, uint64_t* ix, uint64_t* iy,
                                      uint64_t* iz, void* stream);

/* encode_points(x, y, z, level) (_ckernels.pyx:85-104): truncating f64
 * quantisation `(long long)(x * 2^level)` with an upper clamp to 2^level-1,
 * then bit interleave.  x/y/z are strided by *_stride ELEMENTS (so a column
 * of an (N,3) C array has stride 3).  Bit-identical to the compiled backend
 * for every finite or non-finite input. */
FMMB_API fmmb_status fmmb_encode_points(fmmb_handle_t h, const double* x,
                               int64_t x_stride, const double* y,
                               int64_t y_stride, const double* z,
                               int64_t z_stride, int64_t n, int level,
                               uint64_t* out, void* stream);

/* assign_box_ranks(boxes, nbins) (_ckernels.pyx:107-119): dense occupancy
 * histogram `bins[nbins]` and arrival-order rank of each point in its box.
 * Requires boxes[i] < nbins (FMMB_ERR_DOMAIN otherwise; the reference indexes
 * out of bounds there). `bins` and `ranks` are caller-allocated. */
FMMB_API fmmb_status fmmb_assign_box_ranks(fmmb_handle_t h, const uint64_t* boxes,
                                  int64_t n, int64_t nbins, int64_t* bins,
                                  int64_t* ranks, void* stream);

/* adjacent_segments(recv_boxes, src_boxes, level) (_ckernels.pyx:140-202):
 * per receiver box, ranks into src_boxes (ascending, lower_bound semantics)
 * of the in-grid 3x3x3 window members present in src_boxes.
 * `bookmark` (nr+1, caller-allocated); the flat list is allocated through
 * `alloc` with exactly *total entries. */
FMMB_API fmmb_status fmmb_adjacent_segments(fmmb_handle_t h, const uint64_t* recv,
                                   int64_t nr, const uint64_t* src, int64_t ns,
                                   int level, int64_t* bookmark,
                                   fmmb_alloc_fn alloc, void* ctx,
                                   int64_t** list, int64_t* total,
                                   void* stream);

/* stencil_segments(recv_boxes, src_boxes, level) (_ckernels.pyx:205-287):
 * per receiver box, ranks into src_boxes of the children of the parent's
 * 3x3x3 window that are not in the box's own 3x3x3 window, ascending, and
 * the i16 offset codes (dx+3)+7(dy+3)+49(dz+3).  Empty lists for level < 2. */
FMMB_API fmmb_status fmmb_stencil_segments(fmmb_handle_t h, const uint64_t* recv,
                                  int64_t nr, const uint64_t* src, int64_t ns,
                                  int level, int64_t* bookmark,
                                  fmmb_alloc_fn alloc, void* ctx,
                                  int64_t** ranks, int16_t** codes,
                                  int64_t* total, void* stream);

/* propagate_to_parents(boxes) (lists.py:103-105): ascending unique of
 * boxes >> 3 for an ascending input.  `out` has capacity n; *count written. */
FMMB_API fmmb_status fmmb_propagate_to_parents(fmmb_handle_t h, const uint64_t* boxes,
                                      int64_t n, uint64_t* out,
                                      int64_t* count, void* stream);

/* exclusive_scan(values) (scan.py:25-73): out[i] = sum(values[:i]); *total.
 * Values must be non-negative (FMMB_ERR_DOMAIN otherwise). */
FMMB_API fmmb_status fmmb_exclusive_scan_i64(fmmb_handle_t h, const int64_t* values,
                                    int64_t n, int64_t* out, int64_t* total,
                                    void* stream);

/* build_bookmarks(bins) (pseudosort.py:68-78): bookmarks (k+1,) = [0,
 * cumsum(bins[nz])] and the non-empty indices nz (k,) of a dense histogram,
 * both allocated through `alloc`.  Negative counts raise FMMB_ERR_DOMAIN. */
FMMB_API fmmb_status fmmb_build_bookmarks(fmmb_handle_t h, const int64_t* bins,
                                 int64_t nbins, fmmb_alloc_fn alloc, void* ctx,
                                 int64_t** bookmarks, uint64_t** non_empty,
                                 int64_t* k, void* stream);

/* Workload driver (c4 dynamic rebuild; not a reference entry point):
 * x[i] <- mod(x[i] + N(0, scale^2), 1.0) in place, np.mod's convention,
 * normals from Philox4x32-10 keyed by (seed, step). */
FMMB_API fmmb_status fmmb_perturb(fmmb_handle_t h, double* x, int64_t n, uint64_t seed,
                         uint64_t step, double scale, void* stream);

/* --------------------------------------------------------- build API level */

/* One sorted point set, reference layout (pseudosort.py:81-102). */
typedef struct fmmb_point_set {
  double* points;      /* (n, 3) f64, grouped by box, boxes ascending */
  double* charges;     /* (n,) f64 or NULL (receivers)                 */
  int64_t* permutation;/* (n,) sorted position -> original position    */
  int64_t* bookmarks;  /* (k + 1,)                                      */
  uint64_t* non_empty; /* (k,) ascending Morton indices at max level    */
  uint64_t* boxes;     /* (n,) Morton index of each sorted point        */
  int64_t n;
  int64_t k;
} fmmb_point_set;

/* The whole FmmStructures bundle (lists.py:58-66).  Per-level arrays are
 * indexed by level 0..FMMB_MAX_LEVEL; entries outside the reference's dicts
 * (directory levels < 2 except max_level, stencil levels < 2) are NULL. */
typedef struct fmmb_structures {
  int32_t max_level;
  int32_t _pad;
  fmmb_point_set src;
  fmmb_point_set recv;
  /* NeighborTable (lists.py:21-30) */
  int64_t* neighbor_bookmark; /* (k_recv + 1,) */
  int64_t* neighbor_list;     /* (n_neighbor,) */
  int64_t n_neighbor;
  /* LevelDirectory (lists.py:33-42) */
  uint64_t* dir_src[FMMB_MAX_LEVEL + 1];
  uint64_t* dir_recv[FMMB_MAX_LEVEL + 1];
  int64_t n_dir_src[FMMB_MAX_LEVEL + 1];
  int64_t n_dir_recv[FMMB_MAX_LEVEL + 1];
  /* TranslationStencils (lists.py:45-55) */
  int64_t* st_bookmark[FMMB_MAX_LEVEL + 1]; /* (n_dir_recv[l] + 1,) */
  int64_t* st_ranks[FMMB_MAX_LEVEL + 1];
  int16_t* st_codes[FMMB_MAX_LEVEL + 1];
  int64_t n_st[FMMB_MAX_LEVEL + 1];
  /* device time of each phase, filled only if `timing` events were given */
  int64_t n_launches;
} fmmb_structures;

/* build_all(src_points, src_charges, recv_points, max_level) (lists.py:133-187)
 * src: (n,3) f64 C-contiguous device array; charges: (n,) f64 or NULL;
 * recv: (m,3) f64.  All outputs are allocated through `alloc` and written to
 * *out.  `timing` is NULL or an array of 6 cudaEvent_t recorded at the phase
 * boundaries [start, sorted, directory, counted, write-start, end] (the
 * size read-back sits between `counted` and `write-start`).
 * Errors: FMMB_ERR_CAPACITY for level outside [0,20]; FMMB_ERR_DOMAIN when a
 * point's Morton index falls outside the level grid (negative coordinates:
 * the reference indexes its histogram out of bounds there). */
FMMB_API fmmb_status fmmb_build_all(fmmb_handle_t h, const double* src,
                           const double* charges, int64_t n,
                           const double* recv, int64_t m, int level,
                           fmmb_alloc_fn alloc, void* ctx,
                           fmmb_structures* out, void** timing, void* stream);

/* sort_points(points, charges, max_level) (pseudosort.py:138-151): the sort
 * half of build_all for a single point set.  Outputs allocated via `alloc`. */
FMMB_API fmmb_status fmmb_sort_points(fmmb_handle_t h, const double* points,
                             const double* charges, int64_t n, int level,
                             fmmb_alloc_fn alloc, void* ctx,
                             fmmb_point_set* out, void* stream);

/* reorder(points, charges, bins, boxes, ranks, max_level) (pseudosort.py:
 * 105-135): permutation[offsets[boxes[i]] + ranks[i]] = i with offsets the
 * exclusive scan of bins, then points / charges / boxes gathered through it
 * and the bookmarks of `bins`; every output array allocated through `alloc`.
 * boxes[i] >= nbins or a position outside [0, n) raise FMMB_ERR_DOMAIN. */
FMMB_API fmmb_status fmmb_reorder(fmmb_handle_t h, const double* points,
                         const double* charges, int64_t n, const int64_t* bins,
                         int64_t nbins, const uint64_t* boxes, const int64_t* ranks,
                         int level, fmmb_alloc_fn alloc, void* ctx,
                         fmmb_point_set* out, void* stream);

/* ------------------------------------------- multi-GPU (Morton partition) */
/* The build of one problem across P GPUs (PAPER.md:923-948,
 * partition.py:22-61 for the contiguous-range ownership).  The host drives
 * the collectives between these calls (paper_1301_1704_b200/distributed.py):
 *   fmmb_part_histogram -> all-reduce -> cut bins into P ranges ->
 *   fmmb_part_pack -> all-to-all -> fmmb_dist_sort -> all-reduce (SUM = OR)
 *   of the level-L bitmaps -> fmmb_dist_lists.
 * The concatenation over ranks of every output equals fmmb_build_all on the
 * whole problem. */

/* Histogram of the top `pbits` (<= 14, <= 3L) level-L Morton-key bits over
 * [src | recv] into hist[2^pbits] (u32, device). */
FMMB_API fmmb_status fmmb_part_histogram(fmmb_handle_t h, const double* src, int64_t n,
                                const double* recv, int64_t m, int level, int pbits,
                                uint32_t* hist, void* stream);

/* Stable partition of [src | recv] by destination rank bin_rank[bin] into
 * send buffers grouped by destination (input order kept inside a group):
 * sxyz (n,3), sq (n) or NULL, sgid (n) = gbase_src + local index, rxyz (m,3),
 * rgid (m).  counts (HOST, 2*nranks): points per destination, src then recv. */
FMMB_API fmmb_status fmmb_part_pack(fmmb_handle_t h, const double* src, const double* q,
                           int64_t n, const double* recv, int64_t m, int level, int pbits,
                           const uint32_t* bin_rank, int nranks, int64_t gbase_src,
                           int64_t gbase_recv, double* sxyz, double* sq, int64_t* sgid,
                           double* rxyz, int64_t* rgid, int64_t* counts, void* stream);

/* Sort phase of one rank's owned points (global indices gid_*): sorted
 * point sets with rank-local bookmarks / non-empty keys and permutations in
 * GLOBAL indices, plus the level-L occupancy bitmaps (bmp: 2 * max(1,8^L/64)
 * u64 words, src then recv) for the all-reduce. */
FMMB_API fmmb_status fmmb_dist_sort(fmmb_handle_t h, const double* src, const double* q,
                           int64_t n, const int64_t* gid_src, const double* recv, int64_t m,
                           const int64_t* gid_recv, int level, fmmb_alloc_fn alloc, void* ctx,
                           fmmb_point_set* src_out, fmmb_point_set* recv_out, uint64_t* bmp,
                           void* stream);
/* fmmb_dist_sort returns once the occupancy bitmap (`bmp`) and the box
 * counts are final; its local pass (sorted points, permutation, bookmarks)
 * may still run on the handle's side stream, beside the bitmap all-reduce
 * and fmmb_dist_lists.  fmmb_dist_join orders `stream` after it: call it
 * before reading the sorted point sets. */
FMMB_API fmmb_status fmmb_dist_join(fmmb_handle_t h, void* stream);

/* Lists of one rank from the GLOBAL level-L bitmaps (gbmp, layout as above):
 * receiver rows owned by the key window [key_lo, key_hi) at every level (a
 * box is owned when its first level-L key is), E2/E4 entries as global
 * source ranks, CSR bookmarks starting at 0 (the host adds the offsets of
 * the preceding ranks), owned windows of the level directory (levels 2..L-1).
 * out->recv.k = owned level-L rows. */
FMMB_API fmmb_status fmmb_dist_lists(fmmb_handle_t h, const uint64_t* gbmp, int level,
                            uint64_t key_lo, uint64_t key_hi, fmmb_alloc_fn alloc, void* ctx,
                            fmmb_structures* out, void* stream);

/* Fused pack + exchange over peer memory (multi-GPU without a separate
 * all-to-all).  fmmb_part_counts: counts[set * nranks + r] of this rank's
 * points per destination rank (as fmmb_part_pack reports them), so every
 * rank can size its receive arrays.  fmmb_part_pack_peer: the same stable
 * partition, each point stored directly into destination r's arrays
 * sxyz[r] (n_r x 3), sq[r] (or NULL), sgid[r], rxyz[r], rgid[r] -- device
 * pointers valid on this device (peer-mapped with CUDA IPC / P2P, or the
 * same device) -- starting at element soff[r] / roff[r] (this rank's block
 * at r: the counts of lower source ranks).  Ends with a system-scope fence;
 * the caller synchronises the stream and barriers before the receivers read. */
FMMB_API fmmb_status fmmb_part_counts(fmmb_handle_t h, const double* src, int64_t n,
                             const double* recv, int64_t m, int level, int pbits,
                             const uint32_t* bin_rank, int nranks, int64_t* counts,
                             void* stream);
FMMB_API fmmb_status fmmb_part_pack_peer(fmmb_handle_t h, const double* src, const double* q,
                                int64_t n, const double* recv, int64_t m, int level, int pbits,
                                const uint32_t* bin_rank, int nranks, int64_t gbase_src,
                                int64_t gbase_recv, double* const* sxyz, double* const* sq,
                                int64_t* const* sgid, double* const* rxyz,
                                int64_t* const* rgid, const int64_t* soff, const int64_t* roff,
                                void* stream);

/* ------------------------------------------- consumers of the structures */

/* near_field(sx, sy, sz, sq, src_bookmark, nbr_bookmark, nbr_list, rx, ry,
 * rz, recv_bookmark) (_ckernels.pyx:290-323; caller fmm.py:173-190):
 * phi[r] for every receiver r of receiver box j = sum over the sources of
 * the boxes nbr_list[nbr_bookmark[j]:nbr_bookmark[j+1]] (segment order,
 * points in sorted order) of q/|r - s|, skipping coincident pairs.
 * Bit-identical to the compiled backend (sequential f64 sum, IEEE sqrt and
 * divide, no contraction).  Coordinates strided by *_stride ELEMENTS; q may
 * be NULL (unit charges).  Receivers outside every box get 0.
 * nbr_bookmark and recv_bookmark both have n_recv_boxes + 1 entries. */
FMMB_API fmmb_status fmmb_near_field(fmmb_handle_t h, const double* sx, int64_t sx_stride,
                            const double* sy, int64_t sy_stride, const double* sz,
                            int64_t sz_stride, const double* q, int64_t ns,
                            const int64_t* src_bookmark, int64_t n_src_boxes,
                            const int64_t* nbr_bookmark, const int64_t* nbr_list,
                            int64_t n_nbr, const double* rx, int64_t rx_stride,
                            const double* ry, int64_t ry_stride, const double* rz,
                            int64_t rz_stride, int64_t nr, const int64_t* recv_bookmark,
                            int64_t n_recv_boxes, double* phi, void* stream);

/* direct_potentials(sx, sy, sz, sq, rx, ry, rz) (_ckernels.pyx:326-350;
 * caller fmm.py:21-30 direct_sum): every receiver against every source in
 * source order, same exactness contract as fmmb_near_field. */
FMMB_API fmmb_status fmmb_direct_potentials(fmmb_handle_t h, const double* sx,
                                   int64_t sx_stride, const double* sy, int64_t sy_stride,
                                   const double* sz, int64_t sz_stride, const double* q,
                                   int64_t ns, const double* rx, int64_t rx_stride,
                                   const double* ry, int64_t ry_stride, const double* rz,
                                   int64_t rz_stride, int64_t nr, double* phi, void* stream);

/* classify(node, global_src_boxes, plan) for ONE level (boxtype.py:103-144,
 * stencil owners :63-101): types[i] in {0 DOMESTIC, 1 EXPORT, 2 IMPORT,
 * 3 ROOT, 4 OTHER} of the global non-empty source box boxes[i] at `level`
 * for `node`, given the partition-level owner-unit table box_proc_id
 * (8^partition_level entries, int32).  FMMB_ERR_DOMAIN for level < 2 and
 * for levels the reference cannot resolve to one unit. */
FMMB_API fmmb_status fmmb_classify_boxes(fmmb_handle_t h, const uint64_t* boxes, int64_t n,
                                int level, const int32_t* box_proc_id,
                                int64_t n_units_table, int partition_level,
                                int critical_level, int nodes, int units_per_node, int node,
                                int8_t* types, void* stream);

/* One candidate level of choose_partition (partition.py:74-127): the dense
 * load of `level` (recv_counts of the boxes at from_level summed into their
 * level-`level` ancestors), its inclusive prefix incl, and for k = 0..units
 * bounds[k] (0, searchsorted_left(incl, total*k/units) + 1 capped at 8^level,
 * 8^level) and cum[k] = incl[bounds[k] - 1] (0 for bounds 0).  bounds and cum
 * are caller-allocated (units + 1). */
FMMB_API fmmb_status fmmb_partition_level(fmmb_handle_t h, const uint64_t* recv_boxes,
                                 const int64_t* recv_counts, int64_t n, int from_level,
                                 int level, int64_t total, int units, int64_t* bounds,
                                 int64_t* cum, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FMMB200_H */
