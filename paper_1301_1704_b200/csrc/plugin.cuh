// Kernel-plugin level of libfmmb200: the functions of the reference's
// `fmmkit.backend.kernels` module (_ckernels.pyx / _pykernels.py) on the GPU,
// with arbitrary (not necessarily hierarchical) inputs.  Included by build.cu
// (single translation unit).
#pragma once
#include "common.cuh"
#include "sort.cuh"

namespace fmmb {

// ------------------------------------------------------------ elementwise
__global__ void k_spread(const uint64_t* __restrict__ v, int64_t n, uint64_t* __restrict__ o) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o[i] = dilate3(v[i]);
}
__global__ void k_compact(const uint64_t* __restrict__ v, int64_t n, uint64_t* __restrict__ o) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o[i] = undilate3(v[i]);
}
__global__ void k_interleave(const uint64_t* __restrict__ x, const uint64_t* __restrict__ y,
                             const uint64_t* __restrict__ z, int64_t n,
                             uint64_t* __restrict__ o) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o[i] = morton3(x[i], y[i], z[i]);
}
__global__ void k_deinterleave(const uint64_t* __restrict__ v, int64_t n,
                               uint64_t* __restrict__ x, uint64_t* __restrict__ y,
                               uint64_t* __restrict__ z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = v[i];
    x[i] = undilate3(k);
    y[i] = undilate3(k >> 1);
    z[i] = undilate3(k >> 2);
  }
}
// encode_points on strided columns (_ckernels.pyx:85-104)
__global__ void k_encode_strided(const double* __restrict__ x, int64_t sx,
                                 const double* __restrict__ y, int64_t sy,
                                 const double* __restrict__ z, int64_t sz, int64_t n,
                                 int level, uint64_t* __restrict__ o) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o[i] = encode_point(__ldg(x + i * sx), __ldg(y + i * sy), __ldg(z + i * sz), level);
}

// ------------------------------------------------------------ scans -------
constexpr int kXThreads = 256;
constexpr int kXItems = 8;
constexpr int kXTile = kXThreads * kXItems;

// Single-pass exclusive scan of i64 values (decoupled look-back); flags
// negative inputs (err bit 1) and accumulates an f64 sum for the reference's
// overflow guard (scan.py:16,36-37).
__global__ void __launch_bounds__(kXThreads)
    k_scan_i64(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ out,
               uint64_t* __restrict__ states, uint32_t* __restrict__ counter,
               int64_t* __restrict__ total, double* __restrict__ fsum,
               uint32_t* __restrict__ err) {
  __shared__ int64_t s_tile, s_excl;
  __shared__ uint64_t s_w[kXThreads / 32];
  __shared__ double s_f[kXThreads / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t e0 = tile * kXTile + (int64_t)tid * kXItems;
  int64_t v[kXItems];
  uint64_t c = 0;
  double f = 0.0;
  bool neg = false;
#pragma unroll
  for (int i = 0; i < kXItems; ++i) {
    v[i] = (e0 + i < n) ? in[e0 + i] : 0;
    neg |= v[i] < 0;
    c += (uint64_t)v[i];
    f += (double)v[i];
  }
  if (__any_sync(0xffffffffu, neg) && lane == 0) atomicOr(err, 2u);
  uint64_t wt;
  const uint64_t x = warp_excl_scan<uint64_t>(c, wt);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) f += __shfl_xor_sync(0xffffffffu, f, d);
  if (lane == 0) {
    s_w[warp] = wt;
    s_f[warp] = f;
  }
  __syncthreads();
  uint64_t off = 0, tot = 0;
  double ft = 0.0;
#pragma unroll
  for (int i = 0; i < kXThreads / 32; ++i) {
    off += i < warp ? s_w[i] : 0ull;
    tot += s_w[i];
    ft += s_f[i];
  }
  if (tid == 0) {
    uint64_t* st = states + tile;
    uint64_t excl = 0;
    const uint64_t tv = tot & kStValue;
    if (tile == 0) {
      st_state(st, kStInclusive | tv);
    } else {
      st_state(st, kStAggregate | tv);
      excl = lookback(states, tile, 0, 1) & kStValue;
      st_state(st, kStInclusive | ((excl + tv) & kStValue));
    }
    s_excl = (int64_t)excl;
    atomicAdd(fsum, ft);
    if (e0 + kXTile >= n && tile == (n - 1) / kXTile) *total = (int64_t)(excl + tot);
  }
  __syncthreads();
  int64_t r = s_excl + (int64_t)(x + off);
#pragma unroll
  for (int i = 0; i < kXItems; ++i) {
    if (e0 + i < n) out[e0 + i] = r;
    r += v[i];
  }
}

// Dense histogram (assign_box_ranks bins) with i64 atomics.
__global__ void k_dense_hist(const uint64_t* __restrict__ boxes, int64_t n, int64_t nbins,
                             unsigned long long* __restrict__ bins, uint32_t* __restrict__ err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t b = boxes[i];
    if (b < (uint64_t)nbins) atomicAdd(bins + b, 1ull);
    else atomicOr(err, 1u);
  }
}

// ranks[idx[p]] = p - start[key[p]] from the stable (key, idx) sort.
template <typename KeyT>
__global__ void k_ranks_from_sorted(const KeyT* __restrict__ skeys,
                                    const uint32_t* __restrict__ sidx, int64_t n,
                                    const int64_t* __restrict__ start, int64_t nbins,
                                    int64_t* __restrict__ ranks) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = (uint64_t)skeys[p];
    ranks[sidx[p]] = k < (uint64_t)nbins ? p - start[k] : 0;
  }
}

// --------------------------------------------------- compaction of parents
// propagate_to_parents: heads where (b[i]>>3) != (b[i-1]>>3); flags a
// non-ascending input (err bit 4).
__global__ void __launch_bounds__(kXThreads)
    k_parents(const uint64_t* __restrict__ b, int64_t n, uint64_t* __restrict__ out,
              uint64_t* __restrict__ states, uint32_t* __restrict__ counter,
              int64_t* __restrict__ count, uint32_t* __restrict__ err) {
  __shared__ int64_t s_tile, s_excl;
  __shared__ uint32_t s_w[kXThreads / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t e0 = tile * kXTile + (int64_t)tid * kXItems;
  uint32_t hmask = 0, c = 0;
  bool unsorted = false;
  uint64_t prev = (e0 > 0 && e0 - 1 < n) ? b[e0 - 1] : 0;
#pragma unroll
  for (int i = 0; i < kXItems; ++i) {
    const int64_t e = e0 + i;
    if (e < n) {
      const uint64_t cur = b[e];
      if (e > 0 && cur < prev) unsorted = true;
      if (e == 0 || (cur >> 3) != (prev >> 3)) {
        hmask |= 1u << i;
        ++c;
      }
      prev = cur;
    }
  }
  if (__any_sync(0xffffffffu, unsorted) && lane == 0) atomicOr(err, 4u);
  uint32_t wt;
  const uint32_t x = warp_excl_scan(c, wt);
  if (lane == 0) s_w[warp] = wt;
  __syncthreads();
  uint32_t off = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < kXThreads / 32; ++i) {
    off += i < warp ? s_w[i] : 0u;
    tot += s_w[i];
  }
  if (tid == 0) {
    uint64_t* st = states + tile;
    uint64_t excl = 0;
    if (tile == 0) {
      st_state(st, kStInclusive | tot);
    } else {
      st_state(st, kStAggregate | tot);
      excl = lookback(states, tile, 0, 1);
      st_state(st, kStInclusive | (excl + tot));
    }
    s_excl = (int64_t)excl;
    if (tile == (n - 1) / kXTile) *count = (int64_t)(excl + tot);
  }
  __syncthreads();
  int64_t j = s_excl + x + off;
#pragma unroll
  for (int i = 0; i < kXItems; ++i)
    if ((hmask >> i) & 1u) out[j++] = b[e0 + i] >> 3;
}

// ------------------------------------------------ sorted-search list kernels
__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* __restrict__ a, int64_t n,
                                                   uint64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Sorted 3x3x3 in-grid window of box `b` at `level` across the warp:
// lane i < cnt holds the i-th smallest key (others ~0).
__device__ __forceinline__ uint64_t sorted_window(uint64_t b, int level) {
  const int lane = threadIdx.x & 31;
  const int64_t ng = 1ll << level;
  const int64_t x = (int64_t)undilate3(b), y = (int64_t)undilate3(b >> 1),
                z = (int64_t)undilate3(b >> 2);
  uint64_t k = ~0ull;
  if (lane < 27) {
    const int64_t qx = x + lane % 3 - 1, qy = y + (lane / 3) % 3 - 1, qz = z + lane / 9 - 1;
    if (qx >= 0 && qx < ng && qy >= 0 && qy < ng && qz >= 0 && qz < ng)
      k = morton3((uint64_t)qx, (uint64_t)qy, (uint64_t)qz);
  }
#pragma unroll
  for (int s = 2; s <= 32; s <<= 1)
#pragma unroll
    for (int d = s >> 1; d > 0; d >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, k, d);
      const bool want_min = ((lane & d) == 0) == ((lane & s) == 0);
      if (want_min ? (o < k) : (o > k)) k = o;
    }
  return k;
}

// adjacent_segments (_ckernels.pyx:172-202): warp per receiver box, lane per
// sorted window member, lower_bound + equality test (count / write pass).
template <bool WRITE>
__global__ void __launch_bounds__(256)
    k_adjacent(const uint64_t* __restrict__ recv, int64_t nr, const uint64_t* __restrict__ src,
               int64_t ns, int level, int64_t* __restrict__ bm, int64_t* __restrict__ list) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < nr; r += ws) {
    const uint64_t k = sorted_window(__ldg(recv + r), level);
    bool hit = false;
    int64_t pos = 0;
    if (k != ~0ull) {
      pos = lower_bound_u64(src, ns, k);
      hit = pos < ns && __ldg(src + pos) == k;
    }
    const unsigned ball = __ballot_sync(0xffffffffu, hit);
    if (!WRITE) {
      if (lane == 0) bm[r] = __popc(ball);  // count pass: bm is the count array
    } else if (hit) {
      list[bm[r] + __popc(ball & lanemask_lt())] = pos;
    }
  }
}

// stencil_segments (_ckernels.pyx:228-286): warp per receiver box, lane per
// sorted parent-window member; each lane scans src from lower_bound(p<<3)
// while < (p<<3)+8 and keeps the children outside the own window.
template <bool WRITE>
__global__ void __launch_bounds__(256)
    k_stencil(const uint64_t* __restrict__ recv, int64_t nr, const uint64_t* __restrict__ src,
              int64_t ns, int level, int64_t* __restrict__ bm, int64_t* __restrict__ ranks,
              int16_t* __restrict__ codes) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < nr; r += ws) {
    const uint64_t rb = __ldg(recv + r);
    const int64_t cx = (int64_t)undilate3(rb), cy = (int64_t)undilate3(rb >> 1),
                  cz = (int64_t)undilate3(rb >> 2);
    const uint64_t pk = sorted_window(rb >> 3, level - 1);
    int64_t lo = 0, hi = 0;
    if (pk != ~0ull) {
      lo = lower_bound_u64(src, ns, pk << 3);
      hi = lo;
      while (hi < ns && __ldg(src + hi) < (pk << 3) + 8) ++hi;
    }
    const int64_t px = (int64_t)undilate3(pk) << 1, py = (int64_t)undilate3(pk >> 1) << 1,
                  pz = (int64_t)undilate3(pk >> 2) << 1;
    int64_t cnt = 0;
    for (int64_t pos = lo; pos < hi; ++pos) {
      const uint64_t ch = __ldg(src + pos);
      const int64_t dx = (px | (int64_t)(ch & 1)) - cx, dy = (py | (int64_t)((ch >> 1) & 1)) - cy,
                    dz = (pz | (int64_t)((ch >> 2) & 1)) - cz;
      if (dx > 1 || dx < -1 || dy > 1 || dy < -1 || dz > 1 || dz < -1) ++cnt;
    }
    int64_t tot;
    const int64_t excl = warp_excl_scan<int64_t>(cnt, tot);
    if (!WRITE) {
      if (lane == 0) bm[r] = tot;  // count pass: bm is the count array
    } else {
      int64_t w = bm[r] + excl;
      for (int64_t pos = lo; pos < hi; ++pos) {
        const uint64_t ch = __ldg(src + pos);
        const int64_t dx = (px | (int64_t)(ch & 1)) - cx,
                      dy = (py | (int64_t)((ch >> 1) & 1)) - cy,
                      dz = (pz | (int64_t)((ch >> 2) & 1)) - cz;
        if (dx > 1 || dx < -1 || dy > 1 || dy < -1 || dz > 1 || dz < -1) {
          ranks[w] = pos;
          codes[w] = (int16_t)((dx + 3) + 7 * (dy + 3) + 49 * (dz + 3));
          ++w;
        }
      }
    }
  }
}

// build_bookmarks / reorder (pseudosort.py:68-78, 105-135) as device passes.
// k_bm_flags: flags[i] = bins[i] != 0 (np.nonzero), negative bins raise err.
__global__ void k_bm_flags(const int64_t* __restrict__ bins, int64_t n, int64_t* __restrict__ flags,
                           uint32_t* __restrict__ err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = __ldg(bins + i);
    if (b < 0) atomicOr(err, 1u);
    flags[i] = b != 0;
  }
}

// bookmarks[pos+1] = cumsum(bins[nz]) at nz = i, non_empty[pos] = i
__global__ void k_bm_write(const int64_t* __restrict__ bins, const int64_t* __restrict__ excl,
                           const int64_t* __restrict__ pos, int64_t n, int64_t* __restrict__ bm,
                           uint64_t* __restrict__ ne) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = __ldg(bins + i);
    if (b != 0) {
      const int64_t p = __ldg(pos + i);
      bm[p + 1] = __ldg(excl + i) + b;
      ne[p] = (uint64_t)i;
    }
  }
}

// permutation[dense_offsets[boxes[i]] + ranks[i]] = i (pseudosort.py:122-125)
__global__ void k_reorder_perm(const uint64_t* __restrict__ boxes, const int64_t* __restrict__ ranks,
                               const int64_t* __restrict__ start, int64_t n, int64_t nbins,
                               int64_t* __restrict__ perm, uint32_t* __restrict__ err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t b = __ldg(boxes + i);
    if (b >= (uint64_t)nbins) {
      atomicOr(err, 1u);
      continue;
    }
    const int64_t p = __ldg(start + b) + __ldg(ranks + i);
    if (p < 0 || p >= n) {
      atomicOr(err, 2u);
      continue;
    }
    perm[p] = i;
  }
}

// points / charges / boxes gathered through the permutation (pseudosort.py:126-135)
__global__ void k_reorder_gather(const double* __restrict__ pts, const double* __restrict__ q,
                                 const uint64_t* __restrict__ boxes,
                                 const int64_t* __restrict__ perm, int64_t n,
                                 double* __restrict__ pts_out, double* __restrict__ q_out,
                                 uint64_t* __restrict__ boxes_out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = __ldg(perm + j);
    if (i < 0 || i >= n) continue;  // invalid sort index: reported by the host, not read
    pts_out[3 * j] = __ldg(pts + 3 * i);
    pts_out[3 * j + 1] = __ldg(pts + 3 * i + 1);
    pts_out[3 * j + 2] = __ldg(pts + 3 * i + 2);
    if (q) q_out[j] = __ldg(q + i);
    boxes_out[j] = __ldg(boxes + i);
  }
}

}  // namespace fmmb

// ============================================================ host (C ABI)
namespace {

using namespace fmmb;

inline int grid_for(int64_t n, int threads, int num_sms) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), (int64_t)num_sms * 16));
}

struct Workspace {  // one stream-ordered allocation, carved in 256-B slices
  char* base = nullptr;
  size_t off = 0, cap = 0;
  cudaStream_t s;
  explicit Workspace(cudaStream_t st) : s(st) {}
  ~Workspace() {
    if (base) cudaFreeAsync(base, s);
  }
  bool overflow = false;
  bool reserve(size_t bytes) {
    cap = bytes + kSlack;
    return cudaMallocAsync((void**)&base, cap, s) == cudaSuccess;
  }
  template <typename T>
  T* take(int64_t count) {
    T* p = (T*)(base + off);
    off += ((size_t)std::max<int64_t>(count, 1) * sizeof(T) + 255) & ~(size_t)255;
    if (off > cap) {  // programming error: report instead of corrupting memory
      overflow = true;
      off -= ((size_t)std::max<int64_t>(count, 1) * sizeof(T) + 255) & ~(size_t)255;
      return (T*)base;
    }
    return p;
  }
  static constexpr size_t kSlack = 1 << 16;
};

inline size_t slice(int64_t count, size_t sz) {
  return ((size_t)std::max<int64_t>(count, 1) * sz + 255) & ~(size_t)255;
}

// Stable LSD radix sort of (key, index) for u64 keys < 2^key_bits.  Returns
// sorted keys (KeyT) and original indices inside `ws`.
template <typename KeyT>
void sort_pairs(fmmb_handle_t h, Workspace& ws, const uint64_t* kin, int64_t n, int key_bits,
                uint32_t* err, KeyT** ks, uint32_t** vs, int64_t* launches) {
  const int npass = std::max(1, (key_bits + kRadixBits - 1) / kRadixBits);
  const int64_t tiles = ceil_div(n, kSortTile);
  KeyT* ka = ws.take<KeyT>(n);
  KeyT* kb = ws.take<KeyT>(n);
  uint32_t* va = ws.take<uint32_t>(n);
  uint32_t* vb = ws.take<uint32_t>(n);
  uint32_t* hist = ws.take<uint32_t>(npass * kBins);
  uint32_t* tc = ws.take<uint32_t>(kMaxPasses);
  uint64_t* st = ws.take<uint64_t>((int64_t)npass * tiles * kBins);
  cudaMemsetAsync(hist, 0, (size_t)npass * kBins * 4, ws.s);
  cudaMemsetAsync(tc, 0, kMaxPasses * 4, ws.s);
  cudaMemsetAsync(st, 0, (size_t)npass * tiles * kBins * 8, ws.s);
  const uint64_t limit = key_bits >= 64 ? ~0ull : (1ull << key_bits);
  k_keys_hist<KeyT><<<grid_for(n, kSortThreads, h->num_sms), kSortThreads, 0, ws.s>>>(
      kin, n, limit, npass, ka, hist, err);
  ++*launches;
  const size_t smem = onesweep_smem_bytes(sizeof(KeyT));
  for (int ps = 0; ps < npass; ++ps) {
    uint64_t* sp = st + (size_t)ps * tiles * kBins;
    if (ps == 0)
      k_onesweep<KeyT, true><<<(unsigned)tiles, kSortThreads, smem, ws.s>>>(
          ka, nullptr, kb, vb, n, 0, hist, sp, tc);
    else
      k_onesweep<KeyT, false><<<(unsigned)tiles, kSortThreads, smem, ws.s>>>(
          ka, va, kb, vb, n, kRadixBits * ps, hist + ps * kBins, sp, tc + ps);
    ++*launches;
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  *ks = ka;
  *vs = va;
}

inline size_t sort_pairs_bytes(int64_t n, int key_bits, size_t key_size) {
  const int npass = std::max(1, (key_bits + kRadixBits - 1) / kRadixBits);
  const int64_t tiles = ceil_div(n, kSortTile);
  return 2 * slice(n, key_size) + 2 * slice(n, 4) + slice(npass * kBins, 4) +
         slice(kMaxPasses, 4) + slice((int64_t)npass * tiles * kBins, 8);
}

// Exclusive scan of i64 counts into out[0..n), out[n] = total; reads back
// (total, f64 sum, error bits) into the pinned block.
struct ScanResult {
  int64_t total;
  double fsum;
  uint32_t err;
};

bool scan_i64(fmmb_handle_t h, Workspace& ws, const int64_t* in, int64_t n, int64_t* out,
              bool write_total_at_end, ScanResult* res, int64_t* launches) {
  const int64_t tiles = std::max<int64_t>(1, ceil_div(n, kXTile));
  uint64_t* st = ws.take<uint64_t>(tiles);
  uint32_t* ctr = ws.take<uint32_t>(4);
  int64_t* tot = ws.take<int64_t>(1);
  double* fs = ws.take<double>(1);
  uint32_t* err = ws.take<uint32_t>(1);
  cudaMemsetAsync(st, 0, tiles * 8, ws.s);
  cudaMemsetAsync(ctr, 0, 16, ws.s);
  cudaMemsetAsync(tot, 0, 8, ws.s);
  cudaMemsetAsync(fs, 0, 8, ws.s);
  cudaMemsetAsync(err, 0, 4, ws.s);
  if (n > 0) {
    k_scan_i64<<<(unsigned)tiles, kXThreads, 0, ws.s>>>(in, n, out, st, ctr, tot, fs, err);
    ++*launches;
  }
  if (write_total_at_end) cudaMemcpyAsync(out + n, tot, 8, cudaMemcpyDeviceToDevice, ws.s);
  ScanResult* hp = (ScanResult*)h->pinned;
  cudaMemcpyAsync(&hp->total, tot, 8, cudaMemcpyDeviceToHost, ws.s);
  cudaMemcpyAsync(&hp->fsum, fs, 8, cudaMemcpyDeviceToHost, ws.s);
  cudaMemcpyAsync(&hp->err, err, 4, cudaMemcpyDeviceToHost, ws.s);
  if (cudaStreamSynchronize(ws.s) != cudaSuccess) return false;
  *res = *hp;
  return true;
}

fmmb_status cuda_status(fmmb_handle_t h, const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fmmb_fail(h, FMMB_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return FMMB_OK;
}

}  // namespace

#define FMMB_ENTER(h)                                        \
  do {                                                       \
    if (!(h)) return FMMB_ERR_ARG;                           \
    cudaSetDevice((h)->device);                              \
    (h)->launches = 0;                                       \
  } while (0)

extern "C" fmmb_status fmmb_spread_bits(fmmb_handle_t h, const uint64_t* v, int64_t n,
                                        uint64_t* out, void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  if (n > 0) {
    k_spread<<<grid_for(n, 256, h->num_sms), 256, 0, (cudaStream_t)stream>>>(v, n, out);
    h->launches = 1;
  }
  return cuda_status(h, "spread_bits");
}

extern "C" fmmb_status fmmb_compact_bits(fmmb_handle_t h, const uint64_t* v, int64_t n,
                                         uint64_t* out, void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  if (n > 0) {
    k_compact<<<grid_for(n, 256, h->num_sms), 256, 0, (cudaStream_t)stream>>>(v, n, out);
    h->launches = 1;
  }
  return cuda_status(h, "compact_bits");
}

extern "C" fmmb_status fmmb_interleave_coords(fmmb_handle_t h, const uint64_t* ix,
                                              const uint64_t* iy, const uint64_t* iz, int64_t n,
                                              uint64_t* out, void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  if (n > 0) {
    k_interleave<<<grid_for(n, 256, h->num_sms), 256, 0, (cudaStream_t)stream>>>(ix, iy, iz, n,
                                                                                  out);
    h->launches = 1;
  }
  return cuda_status(h, "interleave_coords");
}

extern "C" fmmb_status fmmb_deinterleave_indices(fmmb_handle_t h, const uint64_t* idx, int64_t n,
                                                 uint64_t* ix, uint64_t* iy, uint64_t* iz,
                                                 void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  if (n > 0) {
    k_deinterleave<<<grid_for(n, 256, h->num_sms), 256, 0, (cudaStream_t)stream>>>(idx, n, ix,
                                                                                    iy, iz);
    h->launches = 1;
  }
  return cuda_status(h, "deinterleave_indices");
}

extern "C" fmmb_status fmmb_encode_points(fmmb_handle_t h, const double* x, int64_t xs,
                                          const double* y, int64_t ys, const double* z,
                                          int64_t zs, int64_t n, int level, uint64_t* out,
                                          void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  if (level < 0 || level > kMaxLevel)
    return fmmb_fail(h, FMMB_ERR_CAPACITY, "level %d outside [0, %d]", level, kMaxLevel);
  if (n > 0) {
    k_encode_strided<<<grid_for(n, 256, h->num_sms), 256, 0, (cudaStream_t)stream>>>(
        x, xs, y, ys, z, zs, n, level, out);
    h->launches = 1;
  }
  return cuda_status(h, "encode_points");
}

extern "C" fmmb_status fmmb_assign_box_ranks(fmmb_handle_t h, const uint64_t* boxes, int64_t n,
                                             int64_t nbins, int64_t* bins, int64_t* ranks,
                                             void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  cudaStream_t s = (cudaStream_t)stream;
  if (nbins < 1) return fmmb_fail(h, FMMB_ERR_DOMAIN, "nbins must be positive");
  if (n >= (1ll << 32)) return fmmb_fail(h, FMMB_ERR_CAPACITY, "too many points");
  int key_bits = 1;
  while (key_bits < 64 && (1ull << key_bits) < (uint64_t)nbins) ++key_bits;
  const bool k32 = key_bits <= 32;
  Workspace ws(s);
  const size_t bytes = sort_pairs_bytes(n, key_bits, k32 ? 4 : 8) + slice(nbins, 8) + 1024;
  if (!ws.reserve(bytes)) return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation failed");
  uint32_t* err = ws.take<uint32_t>(1);
  cudaMemsetAsync(err, 0, 4, s);
  cudaMemsetAsync(bins, 0, (size_t)nbins * 8, s);
  int64_t* start = ws.take<int64_t>(nbins);
  if (n > 0) {
    k_dense_hist<<<grid_for(n, 256, h->num_sms), 256, 0, s>>>(
        boxes, n, nbins, (unsigned long long*)bins, err);
    ++h->launches;
  }
  // nbins may exceed the sort key range check: validate via the sort's limit
  ScanResult sr;
  if (!scan_i64(h, ws, bins, nbins, start, false, &sr, &h->launches))
    return cuda_status(h, "assign_box_ranks scan");
  if (n > 0) {
    if (k32) {
      uint32_t* ks;
      uint32_t* vs;
      sort_pairs<uint32_t>(h, ws, boxes, n, key_bits, err, &ks, &vs, &h->launches);
      k_ranks_from_sorted<uint32_t><<<grid_for(n, 256, h->num_sms), 256, 0, s>>>(ks, vs, n, start, nbins, ranks);
    } else {
      uint64_t* ks;
      uint32_t* vs;
      sort_pairs<uint64_t>(h, ws, boxes, n, key_bits, err, &ks, &vs, &h->launches);
      k_ranks_from_sorted<uint64_t><<<grid_for(n, 256, h->num_sms), 256, 0, s>>>(ks, vs, n, start, nbins, ranks);
    }
    ++h->launches;
  }
  uint32_t herr = 0;
  cudaMemcpyAsync(h->pinned, err, 4, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_status(h, "assign_box_ranks");
  herr = *(uint32_t*)h->pinned;
  if (herr) return fmmb_fail(h, FMMB_ERR_DOMAIN, "box index outside [0, nbins)");
  return cuda_status(h, "assign_box_ranks");
}

extern "C" fmmb_status fmmb_exclusive_scan_i64(fmmb_handle_t h, const int64_t* values, int64_t n,
                                               int64_t* out, int64_t* total, void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  cudaStream_t s = (cudaStream_t)stream;
  Workspace ws(s);
  if (!ws.reserve(slice(ceil_div(n, kXTile) + 1, 8) + 8192))
    return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation failed");
  ScanResult sr;
  if (!scan_i64(h, ws, values, n, out, false, &sr, &h->launches))
    return cuda_status(h, "exclusive_scan");
  if (sr.err & 2u) return fmmb_fail(h, FMMB_ERR_DOMAIN, "scan input must be non-negative");
  if (sr.fsum > 4611686018427387904.0)
    return fmmb_fail(h, FMMB_ERR_CAPACITY, "scan total would overflow the 64-bit accumulator");
  if (total) *total = sr.total;
  return cuda_status(h, "exclusive_scan");
}

extern "C" fmmb_status fmmb_propagate_to_parents(fmmb_handle_t h, const uint64_t* boxes,
                                                 int64_t n, uint64_t* out, int64_t* count,
                                                 void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    if (count) *count = 0;
    return FMMB_OK;
  }
  Workspace ws(s);
  if (!ws.reserve(sort_pairs_bytes(n, 64, 8) + slice(n, 8) + slice(ceil_div(n, kXTile), 8) + 8192))
    return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation failed");
  uint64_t* st = ws.take<uint64_t>(ceil_div(n, kXTile));
  uint32_t* ctr = ws.take<uint32_t>(4);
  int64_t* cnt = ws.take<int64_t>(1);
  uint32_t* err = ws.take<uint32_t>(1);
  auto run = [&](const uint64_t* in) {
    cudaMemsetAsync(st, 0, (size_t)ceil_div(n, kXTile) * 8, s);
    cudaMemsetAsync(ctr, 0, 16, s);
    cudaMemsetAsync(err, 0, 4, s);
    k_parents<<<(unsigned)ceil_div(n, kXTile), kXThreads, 0, s>>>(in, n, out, st, ctr, cnt, err);
    ++h->launches;
    cudaMemcpyAsync(h->pinned, cnt, 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync((char*)h->pinned + 8, err, 4, cudaMemcpyDeviceToHost, s);
    return cudaStreamSynchronize(s) == cudaSuccess;
  };
  if (!run(boxes)) return cuda_status(h, "propagate_to_parents");
  if (*(uint32_t*)((char*)h->pinned + 8) & 4u) {
    // not ascending: the reference's np.unique sorts first
    uint64_t* ks;
    uint32_t* vs;
    uint32_t* serr = ws.take<uint32_t>(1);
    cudaMemsetAsync(serr, 0, 4, s);
    sort_pairs<uint64_t>(h, ws, boxes, n, 64, serr, &ks, &vs, &h->launches);
    if (!run(ks)) return cuda_status(h, "propagate_to_parents (sorted)");
  }
  if (count) *count = *(int64_t*)h->pinned;
  return cuda_status(h, "propagate_to_parents");
}

namespace {

template <bool STENCIL>
fmmb_status segments_impl(fmmb_handle_t h, const uint64_t* recv, int64_t nr, const uint64_t* src,
                          int64_t ns, int level, int64_t* bookmark, fmmb_alloc_fn alloc,
                          void* ctx, int64_t** ranks, int16_t** codes, int64_t* total,
                          cudaStream_t s) {
  if (level < 0 || level > kMaxLevel)
    return fmmb_fail(h, FMMB_ERR_CAPACITY, "level %d outside [0, %d]", level, kMaxLevel);
  *ranks = nullptr;
  if (codes) *codes = nullptr;
  *total = 0;
  if (nr == 0 || (STENCIL && level < 2)) {
    cudaMemsetAsync(bookmark, 0, (size_t)(nr + 1) * 8, s);
    return cuda_status(h, "segments");
  }
  Workspace ws(s);
  if (!ws.reserve(slice(nr, 8) + slice(ceil_div(nr, kXTile) + 1, 8) + 8192))
    return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation failed");
  int64_t* cnt = ws.take<int64_t>(nr);
  const int grid = grid_for(nr * 32, 256, h->num_sms);
  if (STENCIL)
    k_stencil<false><<<grid, 256, 0, s>>>(recv, nr, src, ns, level, cnt, nullptr, nullptr);
  else
    k_adjacent<false><<<grid, 256, 0, s>>>(recv, nr, src, ns, level, cnt, nullptr);
  ++h->launches;
  ScanResult sr;
  if (!scan_i64(h, ws, cnt, nr, bookmark, true, &sr, &h->launches))
    return cuda_status(h, "segments scan");
  const int64_t tot = sr.total;
  int64_t* r = (int64_t*)alloc(ctx, (uint64_t)std::max<int64_t>(tot, 1) * 8);
  int16_t* c = nullptr;
  if (STENCIL) c = (int16_t*)alloc(ctx, (uint64_t)std::max<int64_t>(tot, 1) * 2);
  if (!r || (STENCIL && !c)) return fmmb_fail(h, FMMB_ERR_ALLOC, "list allocation failed");
  if (tot > 0) {
    if (STENCIL)
      k_stencil<true><<<grid, 256, 0, s>>>(recv, nr, src, ns, level, bookmark, r, c);
    else
      k_adjacent<true><<<grid, 256, 0, s>>>(recv, nr, src, ns, level, bookmark, r);
    ++h->launches;
  }
  *ranks = r;
  if (codes) *codes = c;
  *total = tot;
  return cuda_status(h, "segments");
}

}  // namespace

extern "C" fmmb_status fmmb_adjacent_segments(fmmb_handle_t h, const uint64_t* recv, int64_t nr,
                                              const uint64_t* src, int64_t ns, int level,
                                              int64_t* bookmark, fmmb_alloc_fn alloc, void* ctx,
                                              int64_t** list, int64_t* total, void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  if (!bookmark || !alloc || !list || !total) return FMMB_ERR_ARG;
  return segments_impl<false>(h, recv, nr, src, ns, level, bookmark, alloc, ctx, list, nullptr,
                              total, (cudaStream_t)stream);
}

extern "C" fmmb_status fmmb_stencil_segments(fmmb_handle_t h, const uint64_t* recv, int64_t nr,
                                             const uint64_t* src, int64_t ns, int level,
                                             int64_t* bookmark, fmmb_alloc_fn alloc, void* ctx,
                                             int64_t** ranks, int16_t** codes, int64_t* total,
                                             void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  if (!bookmark || !alloc || !ranks || !codes || !total) return FMMB_ERR_ARG;
  return segments_impl<true>(h, recv, nr, src, ns, level, bookmark, alloc, ctx, ranks, codes,
                             total, (cudaStream_t)stream);
}


namespace {

// bookmarks + non-empty indices of a dense histogram (shared by
// fmmb_build_bookmarks and fmmb_reorder); `excl` = exclusive scan of bins
fmmb_status bookmarks_impl(fmmb_handle_t h, Workspace& ws, const int64_t* bins, int64_t nbins,
                           const int64_t* excl, fmmb_alloc_fn alloc, void* ctx,
                           int64_t** bookmarks, uint64_t** non_empty, int64_t* k) {
  cudaStream_t s = ws.s;
  int64_t* flags = ws.take<int64_t>(nbins);
  int64_t* pos = ws.take<int64_t>(nbins);
  uint32_t* err = ws.take<uint32_t>(1);
  if (ws.overflow) return fmmb_fail(h, FMMB_ERR_CUDA, "internal: workspace overflow");
  cudaMemsetAsync(err, 0, 4, s);
  k_bm_flags<<<grid_for(nbins, 256, h->num_sms), 256, 0, s>>>(bins, nbins, flags, err);
  ++h->launches;
  ScanResult sr;
  if (!scan_i64(h, ws, flags, nbins, pos, false, &sr, &h->launches))
    return cuda_status(h, "build_bookmarks scan");
  const int64_t K = sr.total;
  int64_t* bm = (int64_t*)alloc(ctx, (uint64_t)(K + 1) * 8);
  uint64_t* ne = (uint64_t*)alloc(ctx, (uint64_t)std::max<int64_t>(K, 1) * 8);
  if (!bm || !ne) return fmmb_fail(h, FMMB_ERR_ALLOC, "bookmark allocation failed");
  cudaMemsetAsync(bm, 0, 8, s);
  k_bm_write<<<grid_for(nbins, 256, h->num_sms), 256, 0, s>>>(bins, excl, pos, nbins, bm, ne);
  ++h->launches;
  *bookmarks = bm;
  *non_empty = ne;
  *k = K;
  return cuda_status(h, "build_bookmarks");
}

}  // namespace

extern "C" fmmb_status fmmb_build_bookmarks(fmmb_handle_t h, const int64_t* bins, int64_t nbins,
                                            fmmb_alloc_fn alloc, void* ctx, int64_t** bookmarks,
                                            uint64_t** non_empty, int64_t* k, void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  if (!alloc || !bookmarks || !non_empty || !k || nbins < 0 || (nbins > 0 && !bins))
    return FMMB_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  *bookmarks = nullptr;
  *non_empty = nullptr;
  *k = 0;
  if (nbins == 0) {
    int64_t* bm = (int64_t*)alloc(ctx, 8);
    uint64_t* ne = (uint64_t*)alloc(ctx, 8);
    if (!bm || !ne) return fmmb_fail(h, FMMB_ERR_ALLOC, "bookmark allocation failed");
    cudaMemsetAsync(bm, 0, 8, s);
    *bookmarks = bm;
    *non_empty = ne;
    return cuda_status(h, "build_bookmarks");
  }
  Workspace ws(s);
  if (!ws.reserve(3 * slice(nbins, 8) + 2 * slice(ceil_div(nbins, kXTile) + 1, 8) + 16384))
    return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation failed");
  int64_t* excl = ws.take<int64_t>(nbins);
  ScanResult sr;
  if (!scan_i64(h, ws, bins, nbins, excl, false, &sr, &h->launches))
    return cuda_status(h, "build_bookmarks scan");
  if (sr.err & 2u) return fmmb_fail(h, FMMB_ERR_DOMAIN, "histogram counts must be non-negative");
  return bookmarks_impl(h, ws, bins, nbins, excl, alloc, ctx, bookmarks, non_empty, k);
}

extern "C" fmmb_status fmmb_reorder(fmmb_handle_t h, const double* points, const double* charges,
                                    int64_t n, const int64_t* bins, int64_t nbins,
                                    const uint64_t* boxes, const int64_t* ranks, int level,
                                    fmmb_alloc_fn alloc, void* ctx, fmmb_point_set* out,
                                    void* stream) {
  FMMB_GUARD(h);
  FMMB_ENTER(h);
  if (!alloc || !out || n < 0 || nbins < 1 || !bins || (n > 0 && (!points || !boxes || !ranks)))
    return FMMB_ERR_ARG;
  (void)level;
  cudaStream_t s = (cudaStream_t)stream;
  memset(out, 0, sizeof(*out));
  Workspace ws(s);
  if (!ws.reserve(3 * slice(nbins, 8) + 2 * slice(ceil_div(nbins, kXTile) + 1, 8) + 16384))
    return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation failed");
  int64_t* excl = ws.take<int64_t>(nbins);
  uint32_t* err = ws.take<uint32_t>(1);
  cudaMemsetAsync(err, 0, 4, s);
  ScanResult sr;
  if (!scan_i64(h, ws, bins, nbins, excl, false, &sr, &h->launches))
    return cuda_status(h, "reorder scan");
  if (sr.err & 2u) return fmmb_fail(h, FMMB_ERR_DOMAIN, "histogram counts must be non-negative");
  const size_t nn = (size_t)std::max<int64_t>(n, 1);
  double* pts_out = (double*)alloc(ctx, nn * 24);
  double* q_out = charges ? (double*)alloc(ctx, nn * 8) : nullptr;
  int64_t* perm = (int64_t*)alloc(ctx, nn * 8);
  uint64_t* bx_out = (uint64_t*)alloc(ctx, nn * 8);
  if (!pts_out || (charges && !q_out) || !perm || !bx_out)
    return fmmb_fail(h, FMMB_ERR_ALLOC, "reorder output allocation failed");
  if (n > 0) {
    cudaMemsetAsync(perm, 0xFF, (size_t)n * 8, s);  // unset positions stay -1 (never gathered)
    k_reorder_perm<<<grid_for(n, 256, h->num_sms), 256, 0, s>>>(boxes, ranks, excl, n, nbins,
                                                                  perm, err);
    k_reorder_gather<<<grid_for(n, 256, h->num_sms), 256, 0, s>>>(points, charges, boxes, perm,
                                                                    n, pts_out, q_out, bx_out);
    h->launches += 2;
  }
  cudaMemcpyAsync(h->pinned, err, 4, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_status(h, "reorder");
  const uint32_t herr = *(uint32_t*)h->pinned;
  if (herr & 1u) return fmmb_fail(h, FMMB_ERR_DOMAIN, "box index outside [0, nbins)");
  if (herr & 2u) return fmmb_fail(h, FMMB_ERR_DOMAIN, "sort index position outside [0, n)");
  int64_t* bm = nullptr;
  uint64_t* ne = nullptr;
  int64_t K = 0;
  const fmmb_status st = bookmarks_impl(h, ws, bins, nbins, excl, alloc, ctx, &bm, &ne, &K);
  if (st != FMMB_OK) return st;
  out->points = pts_out;
  out->charges = q_out;
  out->permutation = perm;
  out->bookmarks = bm;
  out->non_empty = ne;
  out->boxes = bx_out;
  out->n = n;
  out->k = K;
  return cuda_status(h, "reorder");
}
