// Receiver-load partition plan: choose_partition
// (partition.py:74-127) per candidate level — the dense Morton-ordered load
// of the level (receiver counts of the finest boxes summed into their
// ancestors), its inclusive prefix, and the P*g - 1 cuts
// searchsorted(incl, total*k/units, 'left') + 1 — on the device; the host
// keeps the level loop and the balance test on P*g + 1 bounds.
#pragma once

namespace fmmb {
namespace {

__global__ void __launch_bounds__(256)
    k_plan_loads(const uint64_t* __restrict__ boxes, const int64_t* __restrict__ counts,
                 int64_t n, int shift, unsigned long long* __restrict__ dense) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    atomicAdd(dense + (boxes[i] >> shift), (unsigned long long)counts[i]);
}

// bounds[0] = 0, bounds[k] = min(searchsorted_left(incl, total*k/units) + 1, nb)
// for 0 < k < units, bounds[units] = nb (non-decreasing by construction, so
// the reference's running max is the identity); cum[k] = incl[bounds[k]-1]
__global__ void __launch_bounds__(256)
    k_plan_cuts(const int64_t* __restrict__ incl, int64_t nb, int64_t total, int units,
                int64_t* __restrict__ bounds, int64_t* __restrict__ cum) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > units) return;
  if (k == 0 || k == units) {
    const int64_t b = k == 0 ? 0 : nb;
    bounds[k] = b;
    cum[k] = b > 0 ? incl[b - 1] : 0;
    return;
  }
  // numpy: total * arange(1, units, dtype=float64) / units
  const double target = __ddiv_rn(__dmul_rn((double)total, (double)k), (double)units);
  int64_t lo = 0, hi = nb;  // first i with (double)incl[i] >= target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((double)incl[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  const int64_t b = lo + 1 < nb ? lo + 1 : nb;
  bounds[k] = b;
  cum[k] = incl[b - 1];
}

}  // namespace
}  // namespace fmmb

extern "C" fmmb_status fmmb_partition_level(fmmb_handle_t h, const uint64_t* recv_boxes,
                                            const int64_t* recv_counts, int64_t n,
                                            int from_level, int level, int64_t total, int units,
                                            int64_t* bounds, int64_t* cum, void* stream) {
  FMMB_GUARD(h);
  using namespace fmmb;
  FMMB_ENTER(h);
  cudaStream_t s = (cudaStream_t)stream;
  if (level < 0 || level > from_level || from_level > kMaxLevel || units < 1)
    return fmmb_fail(h, FMMB_ERR_DOMAIN, "partition_level: bad levels / units");
  const int64_t nb = 1ll << (3 * level);
  Workspace ws(s);
  if (!ws.reserve(slice(nb, 8) + slice(nb + 1, 8) + slice(ceil_div(nb, kXTile) + 1, 8) + 8192))
    return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation failed");
  int64_t* dense = ws.take<int64_t>(nb);
  int64_t* ex = ws.take<int64_t>(nb + 1);  // exclusive prefix + total: incl = ex + 1
  cudaMemsetAsync(dense, 0, (size_t)nb * 8, s);
  int64_t launches = 0;
  if (n > 0) {
    k_plan_loads<<<grid_for(n, 256, h->num_sms), 256, 0, s>>>(
        recv_boxes, recv_counts, n, 3 * (from_level - level), (unsigned long long*)dense);
    ++launches;
  }
  ScanResult sr;
  if (!scan_i64(h, ws, dense, nb, ex, true, &sr, &launches))
    return cuda_status(h, "partition_level scan");
  k_plan_cuts<<<(units + 256) / 256, 256, 0, s>>>(ex + 1, nb, total, units, bounds, cum);
  h->launches = launches + 1;
  return cuda_status(h, "partition_level");
}
