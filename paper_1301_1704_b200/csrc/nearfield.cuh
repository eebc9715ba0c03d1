// Near-field direct sums on the built structures: the
// first consumer of the E2 lists and the sorted point sets, kept on device.
//
//   near_field(...)        _ckernels.pyx:290-323 (fmm.py:173-190 caller)
//   direct_potentials(...) _ckernels.pyx:326-350 (fmm.py:21-30 caller)
//
// Bit-exactness contract (the compiled backend): per receiver,
//   acc = 0; for every source s in neighbour-segment order:
//     dist = sqrt(dx*dx + dy*dy + dz*dz); if (dist != 0) acc += q[s] / dist
// with IEEE round-to-nearest on every operation and no contraction (gcc -O3
// on x86-64 without -march emits no FMA).  Here every operation is an
// explicit _rn intrinsic, so nvcc cannot fuse or reorder either.
//
// Layout: one warp per receiver box.  The terms q/dist (sqrt + divide: the
// FP64 cost) are computed lane-parallel over 32 sources x up to 32
// receivers into shared memory; lane r then adds row r in source order, so
// the FP64 pipe runs full-width for the expensive part and the sums keep the
// reference's sequential order.  Boxes are handed out by an atomic counter
// (clustered inputs have very uneven boxes).
#pragma once

namespace fmmb {
namespace {

constexpr int kNfWarps = 8;
constexpr int kNfRow = 33;  // padded term row (doubles): conflict-light column reads

struct NfArgs {
  const double *sx, *sy, *sz, *q;
  int64_t sxs, sys, szs;
  const int64_t* sbm;  // src bookmarks (K_s + 1)
  const int64_t* nbm;  // neighbour bookmarks (K_r + 1)
  const int64_t* nlist;
  const double *rx, *ry, *rz;
  int64_t rxs, rys, rzs;
  const int64_t* rbm;  // recv bookmarks (K_r + 1)
  int64_t kr;
  double* phi;
};

template <int RG>
struct NfWarp {
  double terms[RG * kNfRow];
  double rx[RG], ry[RG], rz[RG];
  int64_t sstart[32];
  int64_t cex[32];  // exclusive prefix of segment lengths
  int64_t cin[32];  // inclusive
};

__device__ __forceinline__ double nf_term(double rx, double ry, double rz, double sx, double sy,
                                          double sz, double q) {
  const double dx = __dsub_rn(rx, sx);
  const double dy = __dsub_rn(ry, sy);
  const double dz = __dsub_rn(rz, sz);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  const double dist = __dsqrt_rn(d2);
  // acc + 0.0 == acc for every acc the sum can reach (it starts at +0 and
  // never becomes -0), so a skipped pair may contribute +0.
  return dist != 0.0 ? __ddiv_rn(q, dist) : 0.0;
}

template <int RG>
__global__ void __launch_bounds__(kNfWarps * 32)
k_near_field(NfArgs a, unsigned long long* next) {
  extern __shared__ __align__(16) unsigned char nf_smem[];
  const int lane = threadIdx.x & 31;
  NfWarp<RG>& S = reinterpret_cast<NfWarp<RG>*>(nf_smem)[threadIdx.x >> 5];
  for (;;) {
    unsigned long long jj = 0;
    if (lane == 0) jj = atomicAdd(next, 1ull);
    const int64_t j = (int64_t)__shfl_sync(0xffffffffu, jj, 0);
    if (j >= a.kr) break;
    const int64_t r0 = a.rbm[j], r1 = a.rbm[j + 1];
    if (r1 <= r0) continue;
    const int64_t t0 = a.nbm[j], t1 = a.nbm[j + 1];
    for (int64_t g0 = r0; g0 < r1; g0 += RG) {
      const int rg = (int)std::min<int64_t>(RG, r1 - g0);
      if (lane < rg) {
        const int64_t r = g0 + lane;
        S.rx[lane] = a.rx[r * a.rxs];
        S.ry[lane] = a.ry[r * a.rys];
        S.rz[lane] = a.rz[r * a.rzs];
      }
      double acc = 0.0;
      for (int64_t b = t0; b < t1; b += 32) {  // batches of <= 32 neighbour segments
        const int nseg = (int)std::min<int64_t>(32, t1 - b);
        int64_t st = 0, len = 0;
        if (lane < nseg) {
          const int64_t v = a.nlist[b + lane];
          st = a.sbm[v];
          len = a.sbm[v + 1] - st;
        }
        int64_t inc = len;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int64_t o = __shfl_up_sync(0xffffffffu, inc, d);
          if (lane >= d) inc += o;
        }
        S.sstart[lane] = st;
        S.cex[lane] = inc - len;
        S.cin[lane] = inc;
        const int64_t total = __shfl_sync(0xffffffffu, inc, 31);
        __syncwarp();
        for (int64_t c = 0; c < total; c += 32) {
          const int64_t f = c + lane;
          const int nv = (int)std::min<int64_t>(32, total - c);
          if (lane < nv) {
            // segment of flat position f: first k with cin[k] > f
            int k = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1)
              if (S.cin[k + step - 1] <= f) k += step;
            const int64_t s = S.sstart[k] + (f - S.cex[k]);
            const double sx = a.sx[s * a.sxs], sy = a.sy[s * a.sys], sz = a.sz[s * a.szs];
            const double q = a.q ? a.q[s] : 1.0;
            double* col = S.terms + lane;
#pragma unroll 4
            for (int r = 0; r < rg; ++r)
              col[r * kNfRow] = nf_term(S.rx[r], S.ry[r], S.rz[r], sx, sy, sz, q);
          }
          __syncwarp();
          if (lane < rg) {
            const double* row = S.terms + lane * kNfRow;
            for (int k = 0; k < nv; ++k) acc = __dadd_rn(acc, row[k]);
          }
          __syncwarp();
        }
      }
      if (lane < rg) a.phi[g0 + lane] = acc;
      __syncwarp();
    }
  }
}

// direct_potentials: every receiver against every source, in source order.
constexpr int kDpThreads = 256;

__global__ void __launch_bounds__(kDpThreads)
k_direct(const double* sx, int64_t sxs, const double* sy, int64_t sys, const double* sz,
         int64_t szs, const double* q, int64_t ns, const double* rx, int64_t rxs,
         const double* ry, int64_t rys, const double* rz, int64_t rzs, int64_t nr,
         double* phi) {
  __shared__ double tx[kDpThreads], ty[kDpThreads], tz[kDpThreads], tq[kDpThreads];
  for (int64_t base = (int64_t)blockIdx.x * kDpThreads; base < nr;
       base += (int64_t)gridDim.x * kDpThreads) {
    const int64_t i = base + threadIdx.x;
    const bool live = i < nr;
    const double x = live ? rx[i * rxs] : 0.0, y = live ? ry[i * rys] : 0.0,
                 z = live ? rz[i * rzs] : 0.0;
    double acc = 0.0;
    for (int64_t k0 = 0; k0 < ns; k0 += kDpThreads) {
      const int nk = (int)std::min<int64_t>(kDpThreads, ns - k0);
      __syncthreads();
      if (threadIdx.x < nk) {
        const int64_t k = k0 + threadIdx.x;
        tx[threadIdx.x] = sx[k * sxs];
        ty[threadIdx.x] = sy[k * sys];
        tz[threadIdx.x] = sz[k * szs];
        tq[threadIdx.x] = q ? q[k] : 1.0;
      }
      __syncthreads();
#pragma unroll 4
      for (int k = 0; k < nk; ++k) acc = __dadd_rn(acc, nf_term(x, y, z, tx[k], ty[k], tz[k], tq[k]));
    }
    if (live) phi[i] = acc;
  }
}

}  // namespace
}  // namespace fmmb

extern "C" fmmb_status fmmb_near_field(fmmb_handle_t h, const double* sx, int64_t sxs,
                                       const double* sy, int64_t sys, const double* sz,
                                       int64_t szs, const double* q, int64_t ns,
                                       const int64_t* src_bookmark, int64_t n_src_boxes,
                                       const int64_t* nbr_bookmark, const int64_t* nbr_list,
                                       int64_t n_nbr, const double* rx, int64_t rxs,
                                       const double* ry, int64_t rys, const double* rz,
                                       int64_t rzs, int64_t nr, const int64_t* recv_bookmark,
                                       int64_t n_recv_boxes, double* phi, void* stream) {
  FMMB_GUARD(h);
  using namespace fmmb;
  FMMB_ENTER(h);
  cudaStream_t s = (cudaStream_t)stream;
  if (ns < 0 || nr < 0 || n_src_boxes < 0 || n_recv_boxes < 0 || n_nbr < 0)
    return fmmb_fail(h, FMMB_ERR_DOMAIN, "near_field: negative size");
  if (nr > 0) cudaMemsetAsync(phi, 0, (size_t)nr * 8, s);
  if (nr == 0 || n_recv_boxes == 0 || n_nbr == 0 || ns == 0) return cuda_status(h, "near_field");
  Workspace ws(s);
  if (!ws.reserve(256)) return fmmb_fail(h, FMMB_ERR_CUDA, "workspace allocation failed");
  unsigned long long* next = ws.take<unsigned long long>(1);
  cudaMemsetAsync(next, 0, 8, s);
  NfArgs a{sx, sy, sz, q, sxs, sys, szs, src_bookmark, nbr_bookmark, nbr_list,
           rx, ry, rz, rxs, rys, rzs, recv_bookmark, n_recv_boxes, phi};
  const char* rg_env = getenv("FMMB_NF_RG");
  const int rgmax = rg_env ? atoi(rg_env) : 16;
  auto launch = [&](auto kern, size_t smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNfWarps * 32, smem);
    const int64_t want = ceil_div(n_recv_boxes, kNfWarps);
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>(want, (int64_t)h->num_sms * std::max(per_sm, 1)));
    kern<<<grid, kNfWarps * 32, smem, s>>>(a, next);
  };
  if (rgmax == 32)
    launch(k_near_field<32>, sizeof(NfWarp<32>) * kNfWarps);
  else if (rgmax == 8)
    launch(k_near_field<8>, sizeof(NfWarp<8>) * kNfWarps);
  else
    launch(k_near_field<16>, sizeof(NfWarp<16>) * kNfWarps);
  h->launches = 1;
  return cuda_status(h, "near_field");
}

extern "C" fmmb_status fmmb_direct_potentials(fmmb_handle_t h, const double* sx, int64_t sxs,
                                              const double* sy, int64_t sys, const double* sz,
                                              int64_t szs, const double* q, int64_t ns,
                                              const double* rx, int64_t rxs, const double* ry,
                                              int64_t rys, const double* rz, int64_t rzs,
                                              int64_t nr, double* phi, void* stream) {
  FMMB_GUARD(h);
  using namespace fmmb;
  FMMB_ENTER(h);
  cudaStream_t s = (cudaStream_t)stream;
  if (ns < 0 || nr < 0) return fmmb_fail(h, FMMB_ERR_DOMAIN, "direct_potentials: negative size");
  if (nr == 0) return FMMB_OK;
  k_direct<<<grid_for(nr, kDpThreads, h->num_sms), kDpThreads, 0, s>>>(
      sx, sxs, sy, sys, sz, szs, q, ns, rx, rxs, ry, rys, rz, rzs, nr, phi);
  h->launches = 1;
  return cuda_status(h, "direct_potentials");
}
