// C-ABI entry points of the multi-GPU (Morton-range partitioned) build.
// Included by build.cu after build_impl and the plugin helpers.  The host
// (paper_1301_1704_b200/distributed.py) interleaves them with its
// collectives: histogram -> all-reduce -> pack -> all-to-all -> dist_sort ->
// all-reduce of the level-L occupancy bitmaps -> dist_lists.
#include "dist.cuh"

extern "C" fmmb_status fmmb_part_histogram(fmmb_handle_t h, const double* src, int64_t n,
                                           const double* recv, int64_t m, int level, int pbits,
                                           uint32_t* hist, void* stream) {
  FMMB_GUARD(h);
  if (!h || !hist) return FMMB_ERR_ARG;
  if (level < 1 || level > kMaxLevel)
    return fmmb_fail(h, FMMB_ERR_CAPACITY, "max_level %d outside [1, %d]", level, kMaxLevel);
  if (pbits < 1 || pbits > kPartMaxBits || pbits > 3 * level)
    return fmmb_fail(h, FMMB_ERR_ARG, "partition bits %d outside [1, min(%d, 3L)]", pbits,
                     kPartMaxBits);
  cudaSetDevice(h->device);
  h->launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  Workspace ws(s);
  if (!ws.reserve(256)) return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation failed");
  uint32_t* err = ws.take<uint32_t>(1);
  cudaMemsetAsync(err, 0, 4, s);
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) << pbits, s);
  if (n + m > 0) {
    const int grid =
        (int)std::min<int64_t>(ceil_div(n + m, kPartHistThreads), (int64_t)h->num_sms * 2);
    k_part_hist<<<grid, kPartHistThreads, sizeof(uint32_t) << pbits, s>>>(src, n, recv, m, level,
                                                                       pbits, hist, err);
    ++h->launches;
  }
  uint32_t* hp = (uint32_t*)h->pinned;
  cudaMemcpyAsync(hp, err, 4, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_status(h, "part_histogram");
  if (*hp)
    return fmmb_fail(h, FMMB_ERR_DOMAIN,
                     "a point's Morton index lies outside the level-%d grid", level);
  return cuda_status(h, "part_histogram");
}

extern "C" fmmb_status fmmb_part_pack(fmmb_handle_t h, const double* src, const double* q,
                                      int64_t n, const double* recv, int64_t m, int level,
                                      int pbits, const uint32_t* bin_rank, int nranks,
                                      int64_t gbase_src, int64_t gbase_recv, double* sxyz,
                                      double* sq, int64_t* sgid, double* rxyz, int64_t* rgid,
                                      int64_t* counts, void* stream) {
  FMMB_GUARD(h);
  if (!h || !bin_rank || !counts) return FMMB_ERR_ARG;
  if (nranks < 1 || nranks > kPartMaxRanks)
    return fmmb_fail(h, FMMB_ERR_ARG, "nranks %d outside [1, %d]", nranks, kPartMaxRanks);
  if (level < 1 || level > kMaxLevel || pbits < 1 || pbits > kPartMaxBits || pbits > 3 * level)
    return fmmb_fail(h, FMMB_ERR_ARG, "invalid level / partition bits");
  cudaSetDevice(h->device);
  h->launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t tot = n + m;
  const int nslots = 2 * nranks;
  const int64_t ntiles = std::max<int64_t>(1, ceil_div(tot, kPartTile));
  Workspace ws(s);
  if (!ws.reserve(2 * slice(nslots * ntiles + 1, 8) + slice(ceil_div(nslots * ntiles, kXTile) + 1, 8) +
                  8192))
    return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation failed");
  int64_t* cnt = ws.take<int64_t>(nslots * ntiles);
  int64_t* off = ws.take<int64_t>(nslots * ntiles + 1);
  cudaMemsetAsync(cnt, 0, (size_t)nslots * ntiles * 8, s);
  if (tot > 0) {
    k_part_count<<<(unsigned)ntiles, kPartThreads, 0, s>>>(src, n, recv, m, level, pbits,
                                                           bin_rank, nranks, cnt, ntiles);
    ++h->launches;
  }
  ScanResult sr;
  if (!scan_i64(h, ws, cnt, nslots * ntiles, off, false, &sr, &h->launches))
    return cuda_status(h, "part_pack scan");
  if (tot > 0) {
    PartOut o{sxyz, sq, sgid, rxyz, rgid, gbase_src, gbase_recv};
    PeerOut none{};
    k_part_scatter<false><<<(unsigned)ntiles, kPartThreads, 0, s>>>(
        src, q, n, recv, m, level, pbits, bin_rank, nranks, off, ntiles, o, none);
    ++h->launches;
  }
  // per-slot totals = column sums of the slot-major count matrix
  int64_t* hp = (int64_t*)h->pinned;
  for (int sl = 0; sl < nslots; ++sl) {
    const int64_t at = (int64_t)sl * ntiles;
    // off[at] is the slot's start; the next slot's start (or the total) ends it
    cudaMemcpyAsync(hp + sl, off + at, 8, cudaMemcpyDeviceToHost, s);
  }
  if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_status(h, "part_pack");
  for (int sl = 0; sl < nslots; ++sl) {
    const int64_t end = sl + 1 < nslots ? hp[sl + 1] : sr.total;
    counts[sl] = end - hp[sl];
  }
  return cuda_status(h, "part_pack");
}

// Counts only (no scatter): counts[slot] for slot = set * nranks + rank, so the
// receivers can size their arrays before the fused pack + exchange.
// mode 0: counts;  mode 1: scatter into peers (PeerOut from the host tables)
static fmmb_status part_pass(fmmb_handle_t h, const double* src, const double* q, int64_t n,
                             const double* recv, int64_t m, int level, int pbits,
                             const uint32_t* bin_rank, int nranks, int64_t gbase_src,
                             int64_t gbase_recv, const PeerOut* peers, int64_t* counts,
                             cudaStream_t s) {
  using namespace fmmb;
  if (!h || !bin_rank) return FMMB_ERR_ARG;
  if (nranks < 1 || nranks > kPartMaxRanks)
    return fmmb_fail(h, FMMB_ERR_ARG, "nranks %d outside [1, %d]", nranks, kPartMaxRanks);
  if (level < 1 || level > kMaxLevel || pbits < 1 || pbits > kPartMaxBits || pbits > 3 * level)
    return fmmb_fail(h, FMMB_ERR_ARG, "invalid level / partition bits");
  cudaSetDevice(h->device);
  h->launches = 0;
  const int64_t tot = n + m;
  const int nslots = 2 * nranks;
  const int64_t ntiles = std::max<int64_t>(1, ceil_div(tot, kPartTile));
  Workspace ws(s);
  if (!ws.reserve(2 * slice(nslots * ntiles + 1, 8) +
                  slice(ceil_div(nslots * ntiles, kXTile) + 1, 8) + 8192))
    return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation failed");
  int64_t* cnt = ws.take<int64_t>(nslots * ntiles);
  int64_t* off = ws.take<int64_t>(nslots * ntiles + 1);
  cudaMemsetAsync(cnt, 0, (size_t)nslots * ntiles * 8, s);
  if (tot > 0) {
    k_part_count<<<(unsigned)ntiles, kPartThreads, 0, s>>>(src, n, recv, m, level, pbits,
                                                           bin_rank, nranks, cnt, ntiles);
    ++h->launches;
  }
  ScanResult sr;
  if (!scan_i64(h, ws, cnt, nslots * ntiles, off, false, &sr, &h->launches))
    return cuda_status(h, "part scan");
  if (peers) {
    if (tot > 0) {
      PartOut o{nullptr, nullptr, nullptr, nullptr, nullptr, gbase_src, gbase_recv};
      k_part_scatter<true><<<(unsigned)ntiles, kPartThreads, 0, s>>>(
          src, q, n, recv, m, level, pbits, bin_rank, nranks, off, ntiles, o, *peers);
      ++h->launches;
    }
    return cuda_status(h, "part_pack_peer");
  }
  int64_t* hp = (int64_t*)h->pinned;
  for (int sl = 0; sl < nslots; ++sl)
    cudaMemcpyAsync(hp + sl, off + (int64_t)sl * ntiles, 8, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_status(h, "part_counts");
  for (int sl = 0; sl < nslots; ++sl)
    counts[sl] = (sl + 1 < nslots ? hp[sl + 1] : sr.total) - hp[sl];
  return cuda_status(h, "part_counts");
}

extern "C" fmmb_status fmmb_part_counts(fmmb_handle_t h, const double* src, int64_t n,
                                        const double* recv, int64_t m, int level, int pbits,
                                        const uint32_t* bin_rank, int nranks, int64_t* counts,
                                        void* stream) {
  FMMB_GUARD(h);
  if (!counts) return FMMB_ERR_ARG;
  return part_pass(h, src, nullptr, n, recv, m, level, pbits, bin_rank, nranks, 0, 0, nullptr,
                   counts, (cudaStream_t)stream);
}

extern "C" fmmb_status fmmb_part_pack_peer(fmmb_handle_t h, const double* src, const double* q,
                                           int64_t n, const double* recv, int64_t m, int level,
                                           int pbits, const uint32_t* bin_rank, int nranks,
                                           int64_t gbase_src, int64_t gbase_recv,
                                           double* const* sxyz, double* const* sq,
                                           int64_t* const* sgid, double* const* rxyz,
                                           int64_t* const* rgid, const int64_t* soff,
                                           const int64_t* roff, void* stream) {
  FMMB_GUARD(h);
  using namespace fmmb;
  if (!h || !sxyz || !sgid || !rxyz || !rgid || !soff || !roff) return FMMB_ERR_ARG;
  if (nranks < 1 || nranks > kPartMaxRanks)
    return fmmb_fail(h, FMMB_ERR_ARG, "nranks %d outside [1, %d]", nranks, kPartMaxRanks);
  PeerOut po{};
  for (int d = 0; d < nranks; ++d) {
    po.sxyz[d] = sxyz[d];
    po.sq[d] = sq ? sq[d] : nullptr;
    po.sgid[d] = sgid[d];
    po.rxyz[d] = rxyz[d];
    po.rgid[d] = rgid[d];
    po.soff[d] = soff[d];
    po.roff[d] = roff[d];
  }
  return part_pass(h, src, q, n, recv, m, level, pbits, bin_rank, nranks, gbase_src, gbase_recv,
                   &po, nullptr, (cudaStream_t)stream);
}

extern "C" fmmb_status fmmb_dist_sort(fmmb_handle_t h, const double* src, const double* q,
                                      int64_t n, const int64_t* gid_src, const double* recv,
                                      int64_t m, const int64_t* gid_recv, int level,
                                      fmmb_alloc_fn alloc, void* ctx, fmmb_point_set* src_out,
                                      fmmb_point_set* recv_out, uint64_t* bmp, void* stream) {
  FMMB_GUARD(h);
  fmmb_status st = check_build_args(h, src, n, recv, m, level, alloc, true);
  if (st != FMMB_OK) return st;
  if (!src_out || !recv_out || !bmp || level < 1) return FMMB_ERR_ARG;
  cudaSetDevice(h->device);
  DistSortArgs dsa{gid_src, gid_recv, bmp, true};
  fmmb_structures tmp;
  cudaStream_t s = (cudaStream_t)stream;
  if (sort_key_bits(level) <= 32)
    st = build_impl<uint32_t>(h, src, q, n, recv, m, level, alloc, ctx, &tmp, nullptr, s, false,
                              &dsa);
  else
    st = build_impl<uint64_t>(h, src, q, n, recv, m, level, alloc, ctx, &tmp, nullptr, s, false,
                              &dsa);
  if (st == FMMB_OK) {
    *src_out = tmp.src;
    *recv_out = tmp.recv;
  }
  return st;
}

extern "C" fmmb_status fmmb_dist_join(fmmb_handle_t h, void* stream) {
  FMMB_GUARD(h);
  cudaSetDevice(h->device);
  if (h->side) cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)h->ev_side, 0);
  return cuda_status(h, "dist_join");
}

namespace {

struct DistListsHost {  // pinned read-back of the two synchronisation points
  int64_t ktot[kMaxSegs];
  int64_t seg_totals[kMaxLevel + 1];
  ListsLayout lay;
};

}  // namespace

extern "C" fmmb_status fmmb_dist_lists(fmmb_handle_t h, const uint64_t* gbmp, int level,
                                       uint64_t key_lo, uint64_t key_hi, fmmb_alloc_fn alloc,
                                       void* ctx, fmmb_structures* out, void* stream) {
  FMMB_GUARD(h);
  if (!h || !gbmp || !alloc || !out) return FMMB_ERR_ARG;
  const int L = level;
  if (L < 1 || L > kMaxLevel) return fmmb_fail(h, FMMB_ERR_CAPACITY, "max_level %d", L);
  if (!fmmb_bitmap_ok(L, 0))
    return fmmb_fail(h, FMMB_ERR_CAPACITY, "level %d occupancy bitmaps exceed the budget", L);
  cudaSetDevice(h->device);
  h->launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int stride = L + 1;
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
  int64_t cs_tiles = 1;  // capacity: <= 8^(l-1) parents per level (L <= 9 here)
  for (int l = std::max(1, lists_lmin_host(L)); l <= L; ++l)
    cs_tiles += ceil_div(1ll << (3 * (l - 1)), kCsParents);
  Carver z;
  const size_t o_tc = z.take<uint32_t>(16);
  const size_t o_rst = z.take<uint64_t>(tiles);
  const size_t o_st4 = z.take<uint64_t>(cs_tiles), o_st2 = z.take<uint64_t>(cs_tiles);
  const size_t o_tot = z.take<int64_t>(kMaxSegs + kMaxLevel + 1);
  const size_t o_bmp = z.take<uint64_t>(words);
  const size_t zero_bytes = z.off;
  const size_t o_dir = z.take<uint32_t>(words);
  const size_t o_low = z.take<uint64_t>(2 * 9);
  const size_t o_lay = z.take<ListsLayout>(1);
  char* ws = nullptr;
  if (cudaMallocAsync((void**)&ws, z.off, s) != cudaSuccess)
    return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation of %zu bytes failed", z.off);
  auto W = [&](size_t o) { return (void*)(ws + o); };
  auto fail = [&](fmmb_status st, const char* what) {
    cudaFreeAsync(ws, s);
    return fmmb_fail(h, st, "%s", what);
  };
  uint64_t* bmp = (uint64_t*)W(o_bmp);
  uint32_t* dir = (uint32_t*)W(o_dir);
  uint32_t* tc = (uint32_t*)W(o_tc);
  int64_t* ktot = (int64_t*)W(o_tot);
  int64_t* seg_totals = ktot + kMaxSegs;
  cudaMemsetAsync(ws, 0, zero_bytes, s);
  cudaMemcpyAsync(bmp + rp.word_off[L], gbmp, level_words(L) * 8, cudaMemcpyDeviceToDevice, s);
  cudaMemcpyAsync(bmp + rp.word_off[stride + L], gbmp + level_words(L), level_words(L) * 8,
                  cudaMemcpyDeviceToDevice, s);
  // coarse levels of the global bitmaps
  int l = L;
  while (l >= 1 && level_words(l - 1) > 256) {
    const int64_t nc = level_words(l - 1);
    k_pyramid<<<(unsigned)ceil_div(2 * nc, 256), 256, 0, s>>>(
        bmp + rp.word_off[l], bmp + rp.word_off[l - 1], bmp + rp.word_off[stride + l],
        bmp + rp.word_off[stride + l - 1], nc);
    ++h->launches;
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
    ++h->launches;
  }
  rp.bmp = bmp;
  rp.dir = dir;
  rp.states = (uint64_t*)W(o_rst);
  rp.tile_counter = tc + 0;
  rp.totals = ktot;
  k_rank<<<(unsigned)tiles, kRThreads, 0, s>>>(rp);  // rank directory + totals, no keys yet
  ++h->launches;
  ListsParams lp{};
  lp.level = L;
  lp.key_lo = key_lo;
  lp.key_hi = key_hi;
  lp.ktot = ktot;
  lp.bmp = bmp;
  lp.dir = dir;
  for (int set = 0; set < 2; ++set)
    for (int k = 0; k <= L; ++k) lp.bmp_off[set][k] = rp.word_off[set * stride + k];
  ListsLayout* glay = (ListsLayout*)W(o_lay);
  k_lists_plan<<<1, 32, 0, s>>>(lp, glay);  // windows (no bookmark arrays yet)
  ++h->launches;
  DistListsHost* hp = (DistListsHost*)h->pinned;
  static_assert(sizeof(DistListsHost) <= kPinnedBytes, "pinned block too small");
  cudaMemcpyAsync(hp->ktot, ktot, sizeof(hp->ktot), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&hp->lay, glay, sizeof(ListsLayout), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return fail(FMMB_ERR_CUDA, "dist_lists phase 1");
  const DistListsHost h1 = *hp;

  // ---- arena: full per-level directory keys (levels 2..L-1), CSR bookmarks of owned rows
  Carver a;
  size_t a_dir[2][kMaxLevel + 1] = {}, a_bm[kMaxLevel + 1] = {};
  for (int k = 2; k < L; ++k) {
    a_dir[0][k] = a.take<uint64_t>(h1.ktot[k]);
    a_dir[1][k] = a.take<uint64_t>(h1.ktot[stride + k]);
  }
  const int64_t rows_L = h1.lay.r_hi[L] - h1.lay.r_lo[L];
  a_bm[0] = a.take<int64_t>(rows_L + 1);
  for (int k = 2; k <= L; ++k) a_bm[k] = a.take<int64_t>(h1.lay.r_hi[k] - h1.lay.r_lo[k] + 1);
  char* arena = (char*)alloc(ctx, std::max<size_t>(a.off, 256));
  if (!arena) return fail(FMMB_ERR_ALLOC, "dist_lists: output allocation failed");
  uint64_t* low = (uint64_t*)W(o_low);
  for (int set = 0; set < 2; ++set)
    for (int k = 0; k <= L; ++k) {
      uint64_t* dst = nullptr;
      if (k < L) {
        if (k == 0) dst = low + set * 9;
        else if (k == 1) dst = low + set * 9 + 1;
        else dst = (uint64_t*)(arena + a_dir[set][k]);
      }
      rp.keys_out[set * stride + k] = dst;
    }
  cudaMemsetAsync(rp.states, 0, (size_t)tiles * 8, s);
  rp.tile_counter = tc + 1;
  k_rank<<<(unsigned)tiles, kRThreads, 0, s>>>(rp);  // again, now writing every level's keys
  ++h->launches;
  for (int k = 0; k < L; ++k) lp.rkeys[k] = rp.keys_out[stride + k];
  lp.bm[0] = (int64_t*)(arena + a_bm[0]);
  for (int k = 2; k <= L; ++k) lp.bm[k] = (int64_t*)(arena + a_bm[k]);
  k_lists_plan<<<1, 32, 0, s>>>(lp, glay);
  k_lists_cscan<false><<<(unsigned)std::max<int64_t>(1, h1.lay.tile_off[L + 1]), kLThreads, 0, s>>>(
      lp, glay, (uint64_t*)W(o_st4), (uint64_t*)W(o_st2), tc + 2, seg_totals);
  h->launches += 2;
  cudaMemcpyAsync(hp->seg_totals, seg_totals, sizeof(hp->seg_totals), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return fail(FMMB_ERR_CUDA, "dist_lists phase 2");
  int64_t segt[kMaxLevel + 1];
  memcpy(segt, hp->seg_totals, sizeof(segt));

  Carver b;
  const size_t b_e2 = b.take<int64_t>(segt[0]);
  size_t b_r[kMaxLevel + 1] = {}, b_c[kMaxLevel + 1] = {};
  for (int k = 2; k <= L; ++k) {
    b_r[k] = b.take<int64_t>(segt[k]);
    b_c[k] = b.take<int16_t>(segt[k]);
  }
  char* arena_b = (char*)alloc(ctx, std::max<size_t>(b.off, 256));
  if (!arena_b) return fail(FMMB_ERR_ALLOC, "dist_lists: list allocation failed");
  lp.ranks_out[0] = (int64_t*)(arena_b + b_e2);
  for (int k = 2; k <= L; ++k) {
    lp.ranks_out[k] = (int64_t*)(arena_b + b_r[k]);
    lp.codes_out[k] = (int16_t*)(arena_b + b_c[k]);
  }
  launch_lists_write(h, lp, glay, h1.lay.work_off[L + 1],
                     lists_sparse(L >= 2 ? segt[L] : 0, h1.lay.r_hi[L] - h1.lay.r_lo[L]), s);
  ++h->launches;

  memset(out, 0, sizeof(*out));
  out->max_level = L;
  out->neighbor_bookmark = lp.bm[0];
  out->neighbor_list = lp.ranks_out[0];
  out->n_neighbor = segt[0];
  out->recv.k = rows_L;
  for (int k = 2; k < L; ++k) {  // owned windows of the global per-level directory
    out->dir_recv[k] = (uint64_t*)(arena + a_dir[1][k]) + h1.lay.r_lo[k];
    out->n_dir_recv[k] = h1.lay.r_hi[k] - h1.lay.r_lo[k];
    out->dir_src[k] = (uint64_t*)(arena + a_dir[0][k]) + h1.lay.rs_lo[k];
    out->n_dir_src[k] = h1.lay.rs_hi[k] - h1.lay.rs_lo[k];
  }
  for (int k = 2; k <= L; ++k) {
    out->st_bookmark[k] = lp.bm[k];
    out->st_ranks[k] = lp.ranks_out[k];
    out->st_codes[k] = lp.codes_out[k];
    out->n_st[k] = segt[k];
  }
  cudaFreeAsync(ws, s);
  out->n_launches = h->launches;
  return cuda_status(h, "dist_lists");
}
