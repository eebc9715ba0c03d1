// Multi-GPU partition kernels (the paper's Morton-range
// decomposition; reference: partition.py:22-61 for the
// contiguous-range ownership, exchange.py:183-272 for the distributed build).
//
//   k_part_hist    : histogram of the top `pbits` finest-level key bits of
//                    every point of [src | recv] (one key space for both).
//                    The host all-reduces it and cuts contiguous bin ranges,
//                    so a box never straddles two ranks.
//   k_part_count /
//   k_part_scatter : stable partition of [src | recv] by destination rank
//                    (bin -> rank table) into send buffers ordered by
//                    (set, destination, input index): xyz, q and the global
//                    index travel; keys are recomputed at the destination.
#pragma once
#include "common.cuh"

namespace fmmb {

constexpr int kPartMaxBits = 14;   // histogram bins <= 2^14 (64 KiB of shared counters)
constexpr int kPartMaxRanks = 64;
constexpr int kPartThreads = 256;
constexpr int kPartItems = 4;
constexpr int kPartTile = kPartThreads * kPartItems;  // points per tile, warp = 128 consecutive

__device__ __forceinline__ uint32_t part_bin(const double* src, const double* recv, int64_t n,
                                             int64_t i, int level, int pbits, bool& bad) {
  const double* p = i < n ? src + 3 * i : recv + 3 * (i - n);
  const uint64_t key = encode_point(__ldg(p), __ldg(p + 1), __ldg(p + 2), level);
  const int sbits = 3 * level;
  bad |= key >= (1ull << sbits);
  return (uint32_t)((key & ((1ull << sbits) - 1ull)) >> (sbits - pbits));
}

constexpr int kPartHistThreads = 1024;  // 2 CTAs (64 KiB counters each) fill an SM

__global__ void __launch_bounds__(kPartHistThreads)
    k_part_hist(const double* __restrict__ src, int64_t n, const double* __restrict__ recv,
                int64_t m, int level, int pbits, uint32_t* __restrict__ hist,
                uint32_t* __restrict__ err) {
  extern __shared__ uint32_t s_ph[];
  const int nb = 1 << pbits;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s_ph[b] = 0;
  __syncthreads();
  bool bad = false;
  const int64_t tot = n + m;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&s_ph[part_bin(src, recv, n, i, level, pbits, bad)], 1u);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (s_ph[b]) atomicAdd(&hist[b], s_ph[b]);
}

// destination "slot" of a point: set * nranks + rank
__device__ __forceinline__ int part_slot(const double* src, const double* recv, int64_t n,
                                         int64_t i, int level, int pbits,
                                         const uint32_t* bin_rank, int nranks) {
  bool bad = false;
  const uint32_t bin = part_bin(src, recv, n, i, level, pbits, bad);
  return (i < n ? 0 : nranks) + (int)__ldg(bin_rank + bin);
}

// per-tile counts of each slot, laid out slot-major: cnt[slot * ntiles + tile]
__global__ void __launch_bounds__(kPartThreads)
    k_part_count(const double* __restrict__ src, int64_t n, const double* __restrict__ recv,
                 int64_t m, int level, int pbits, const uint32_t* __restrict__ bin_rank,
                 int nranks, int64_t* __restrict__ cnt, int64_t ntiles) {
  __shared__ uint32_t s_c[2 * kPartMaxRanks];
  const int nslots = 2 * nranks;
  for (int i = threadIdx.x; i < nslots; i += blockDim.x) s_c[i] = 0;
  __syncthreads();
  const int64_t tot = n + m;
  const int64_t base = (int64_t)blockIdx.x * kPartTile;
  for (int k = 0; k < kPartItems; ++k) {
    const int64_t i = base + k * kPartThreads + threadIdx.x;
    const int sl = i < tot ? part_slot(src, recv, n, i, level, pbits, bin_rank, nranks) : -1;
    // warp-aggregated: few destinations, so most lanes share a counter
    const unsigned peers = __match_any_sync(0xffffffffu, sl);
    if (sl >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&s_c[sl], (uint32_t)__popc(peers));
  }
  __syncthreads();
  for (int sl = threadIdx.x; sl < nslots; sl += blockDim.x)
    cnt[(int64_t)sl * ntiles + blockIdx.x] = s_c[sl];
}

// Fused pack + exchange: each point is stored straight into its destination
// rank's receive arrays (peer memory mapped over NVLink; the same device for
// simulated ranks) at that rank's offset for this source rank's block.
struct PeerOut {
  double* sxyz[kPartMaxRanks];
  double* sq[kPartMaxRanks];
  int64_t* sgid[kPartMaxRanks];
  double* rxyz[kPartMaxRanks];
  int64_t* rgid[kPartMaxRanks];
  int64_t soff[kPartMaxRanks];  // element offset of this rank's block at each destination
  int64_t roff[kPartMaxRanks];
};

struct PartOut {
  double* sxyz;   // (n, 3) sources grouped by destination
  double* sq;     // (n,) or null
  int64_t* sgid;  // (n,) global source index
  double* rxyz;   // (m, 3)
  int64_t* rgid;  // (m,)
  int64_t gbase_src, gbase_recv;  // global index of this rank's first src / recv point
};

// Stable scatter: `off` = exclusive scan of cnt (slot-major), so tile t's
// points of slot s start at off[s * ntiles + t]; inside the tile each warp
// owns 128 consecutive points (4 rounds of 32, in order) and ranks lanes
// with match.any; warps are ordered through per-warp slot counts.
template <bool PEER>
__global__ void __launch_bounds__(kPartThreads)
    k_part_scatter(const double* __restrict__ src, const double* __restrict__ q, int64_t n,
                   const double* __restrict__ recv, int64_t m, int level, int pbits,
                   const uint32_t* __restrict__ bin_rank, int nranks,
                   const int64_t* __restrict__ off, int64_t ntiles, const PartOut o,
                   const __grid_constant__ PeerOut po) {
  constexpr int kW = kPartThreads / 32;
  __shared__ uint32_t s_wc[kW][2 * kPartMaxRanks];
  const int nslots = 2 * nranks;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < nslots; i += 32) s_wc[warp][i] = 0;
  __syncwarp();
  const int64_t tot = n + m;
  const int64_t wbase = (int64_t)blockIdx.x * kPartTile + warp * (32 * kPartItems);
  const unsigned lt = lanemask_lt();
  int sl[kPartItems];
  uint32_t rk[kPartItems];
#pragma unroll
  for (int k = 0; k < kPartItems; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    sl[k] = i < tot ? part_slot(src, recv, n, i, level, pbits, bin_rank, nranks) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, sl[k]);
    const int leader = __ffs(peers) - 1;
    uint32_t before = 0;
    if (lane == leader && sl[k] >= 0) {
      before = s_wc[warp][sl[k]];
      s_wc[warp][sl[k]] = before + __popc(peers);
    }
    before = __shfl_sync(0xffffffffu, before, leader);
    __syncwarp();
    rk[k] = before + __popc(peers & lt);
  }
  __syncthreads();
  // warp w's base in slot s = tile offset + counts of warps < w
  for (int i = threadIdx.x; i < nslots; i += blockDim.x) {
    uint32_t run = 0;
    for (int w = 0; w < kW; ++w) {
      const uint32_t c = s_wc[w][i];
      s_wc[w][i] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kPartItems; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    if (sl[k] < 0) continue;
    const int64_t dst = off[(int64_t)sl[k] * ntiles + blockIdx.x] + s_wc[warp][sl[k]] + rk[k];
    if (PEER) {  // position inside the destination's group -> peer arrays
      const int dr = sl[k] % nranks;
      const int64_t j = dst - off[(int64_t)sl[k] * ntiles];
      if (i < n) {
        const double* p = src + 3 * i;
        double* x = po.sxyz[dr] + 3 * (po.soff[dr] + j);
        x[0] = p[0];
        x[1] = p[1];
        x[2] = p[2];
        if (po.sq[dr]) po.sq[dr][po.soff[dr] + j] = q[i];
        po.sgid[dr][po.soff[dr] + j] = o.gbase_src + i;
      } else {
        const double* p = recv + 3 * (i - n);
        double* x = po.rxyz[dr] + 3 * (po.roff[dr] + j);
        x[0] = p[0];
        x[1] = p[1];
        x[2] = p[2];
        po.rgid[dr][po.roff[dr] + j] = o.gbase_recv + (i - n);
      }
      continue;
    }
    if (i < n) {
      const double* p = src + 3 * i;
      o.sxyz[3 * dst] = p[0];
      o.sxyz[3 * dst + 1] = p[1];
      o.sxyz[3 * dst + 2] = p[2];
      if (o.sq) o.sq[dst] = q[i];
      o.sgid[dst] = o.gbase_src + i;
    } else {
      const int64_t d = dst - n;  // recv slots follow all src slots
      const double* p = recv + 3 * (i - n);
      o.rxyz[3 * d] = p[0];
      o.rxyz[3 * d + 1] = p[1];
      o.rxyz[3 * d + 2] = p[2];
      o.rgid[d] = o.gbase_recv + (i - n);
    }
  }
  if (PEER) __threadfence_system();  // peer stores visible before the host-side barrier
}

}  // namespace fmmb
