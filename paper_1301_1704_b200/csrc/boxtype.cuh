// Box-type classification of the global source boxes for the multi-node
// plan (the paper computes it on the GPU, Alg. 6).
// Reference: classify / _stencil_owner_flags (boxtype.py:63-144), a pure
// integer predicate per box: thread per box, the 6x6x6 children of the
// parent's 3x3x3 window minus the box's own 3x3x3 window, owners from the
// partition-level unit table box_proc_id.
#pragma once

namespace fmmb {
namespace {

enum : int8_t { kDomestic = 0, kExport = 1, kImport = 2, kRoot = 3, kOther = 4 };

struct ClassifyArgs {
  const uint64_t* boxes;
  int64_t n;
  int level, l_par, l_crit, nodes, upn, node;
  const int32_t* bpid;  // owner unit of every partition-level box (8^l_par)
  int8_t* out;
};

__global__ void __launch_bounds__(256) k_classify(const ClassifyArgs a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    const uint64_t b = a.boxes[i];
    int8_t t = kDomestic;
    if (a.nodes == 1 || a.level < a.l_crit) {
      t = kDomestic;
    } else if (a.level == a.l_crit) {
      if (a.l_par == a.l_crit) {
        t = __ldg(a.bpid + b) / a.upn == a.node ? kExport : kImport;
      } else {  // the partition-level children of b (boxtype.py:123-133)
        const uint64_t span = 1ull << (3 * (a.l_par - a.l_crit));
        bool has = false, all = true;
        for (uint64_t c = 0; c < span; ++c) {
          const bool m = __ldg(a.bpid + b * span + c) / a.upn == a.node;
          has |= m;
          all &= m;
        }
        t = !has ? kImport : (all ? kExport : kRoot);
      }
    } else {  // boxtype.py:134-141 with _stencil_owner_flags (:63-101)
      const int sh = 3 * (a.level - a.l_par);
      const bool mine = __ldg(a.bpid + (b >> sh)) / a.upn == a.node;
      const int64_t ix = (int64_t)undilate3(b), iy = (int64_t)undilate3(b >> 1),
                    iz = (int64_t)undilate3(b >> 2);
      const int64_t g = 1ll << a.level;
      bool tm = false, to = false;
      for (int dz = -2; dz < 4; ++dz) {
        const int64_t cz = 2 * (iz >> 1) + dz;
        for (int dy = -2; dy < 4; ++dy) {
          const int64_t cy = 2 * (iy >> 1) + dy;
          for (int dx = -2; dx < 4; ++dx) {
            const int64_t cx = 2 * (ix >> 1) + dx;
            const bool near = llabs(cx - ix) <= 1 && llabs(cy - iy) <= 1 && llabs(cz - iz) <= 1;
            if (near || cx < 0 || cx >= g || cy < 0 || cy >= g || cz < 0 || cz >= g) continue;
            const uint64_t cand = morton3((uint64_t)cx, (uint64_t)cy, (uint64_t)cz);
            const bool m = __ldg(a.bpid + (cand >> sh)) / a.upn == a.node;
            tm |= m;
            to |= !m;
          }
        }
      }
      t = mine ? (to ? kExport : kDomestic) : (tm ? kImport : kOther);
    }
    a.out[i] = t;
  }
}

}  // namespace
}  // namespace fmmb

extern "C" fmmb_status fmmb_classify_boxes(fmmb_handle_t h, const uint64_t* boxes, int64_t n,
                                           int level, const int32_t* box_proc_id,
                                           int64_t n_units_table, int partition_level,
                                           int critical_level, int nodes, int units_per_node,
                                           int node, int8_t* types, void* stream) {
  FMMB_GUARD(h);
  using namespace fmmb;
  FMMB_ENTER(h);
  if (level < 2) return fmmb_fail(h, FMMB_ERR_DOMAIN, "octree data start at level 2");
  if (nodes < 1 || units_per_node < 1 || partition_level < 0 || partition_level > kMaxLevel ||
      n_units_table != (1ll << (3 * partition_level)))
    return fmmb_fail(h, FMMB_ERR_DOMAIN, "invalid partition plan");
  const bool typed = nodes > 1 && level >= critical_level;
  if (typed && level != critical_level && level < partition_level)
    return fmmb_fail(h, FMMB_ERR_DOMAIN,
                     "boxes above the partition level have a unit range, not one unit");
  if (typed && level == critical_level && critical_level > partition_level)
    return fmmb_fail(h, FMMB_ERR_DOMAIN, "critical level below the partition level");
  if (n == 0) return FMMB_OK;
  ClassifyArgs a{boxes, n, level, partition_level, critical_level, nodes, units_per_node, node,
                 box_proc_id, types};
  k_classify<<<grid_for(n, 256, h->num_sms), 256, 0, (cudaStream_t)stream>>>(a);
  h->launches = 1;
  return cuda_status(h, "classify_boxes");
}
