// Variants of k_bkt_scatter to locate its bottleneck (not product code).
#include <cstdio>
#include <vector>
#include <random>
#include "../../paper_1301_1704_b200/csrc/bucket.cuh"
using namespace fmmb;
template <bool NARROW, int VAR>
__global__ void __launch_bounds__(kSThreads, 1)
    k_var(const double* __restrict__ src, const double* __restrict__ q,
                  const double* __restrict__ recv, const BucketGeo g, int level,
                  int64_t cta_rows, uint32_t* __restrict__ cursor, double* __restrict__ rec,
                  uint32_t* __restrict__ idx) {
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
    if (is_src && q && (((uintptr_t)(q + base) & 15) || ((rows * 8) & 15))) return false;
    return true;
  };
  auto produce = [&](int k) {  // thread 0 only
    const int st = k % kSStages;
    if (k >= kSStages) mbar_wait(empty + st, (uint32_t)(k / kSStages - 1) & 1u);
    if (stage_tma(k)) {
      const int64_t base = lo + (int64_t)k * kSRows;
      const int rows = stage_rows(k);
      double* xyz = stage_xyz(k);
      const bool with_q = base < n && q;
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
      if (i < n) xyz[3 * kSRows + tid] = q ? __ldg(q + i) : 0.0;
    }
    const uint32_t b = bucket_of(
        encode_any<NARROW>(xyz[3 * tid], xyz[3 * tid + 1], xyz[3 * tid + 2], level, grid) & kmask,
        i >= n, g);
    if (VAR == 1) return (uint32_t)i;
    return atomicAdd(cursor + (size_t)b * kCursorStride, 1u);
  };
  auto store = [&](int k, uint32_t dst) {
    const double* xyz = stage_xyz(k);
    const int64_t i = lo + (int64_t)k * kSRows + tid;
    if (tid < stage_rows(k)) {
      const double w = i < n ? (q ? xyz[3 * kSRows + tid] : 0.0) : __longlong_as_double(i - n);
      if (VAR == 7) asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(rec + 4 * (size_t)dst), "d"(xyz[3 * tid]), "d"(xyz[3 * tid + 1]), "d"(xyz[3 * tid + 2]), "d"(w) : "memory");
      else if (VAR == 8) asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(rec + 4 * (size_t)dst), "d"(xyz[3 * tid]), "d"(xyz[3 * tid + 1]), "d"(xyz[3 * tid + 2]), "d"(w) : "memory");
      else if (VAR == 9) { uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(rec + 4 * (size_t)dst), "d"(xyz[3 * tid]), "d"(xyz[3 * tid + 1]), "d"(xyz[3 * tid + 2]), "d"(w), "l"(pol) : "memory"); }
      else if (VAR == 5) rec[4 * (size_t)dst] = xyz[3 * tid];
      else if (VAR == 6) { reinterpret_cast<double2*>(rec)[2 * (size_t)dst] = make_double2(xyz[3 * tid], xyz[3 * tid + 1]);
                           reinterpret_cast<double2*>(rec)[2 * (size_t)dst + 1] = make_double2(xyz[3 * tid + 2], w); }
      else if (VAR != 2) st_v4f64(rec + 4 * (size_t)dst, xyz[3 * tid], xyz[3 * tid + 1], xyz[3 * tid + 2], w);
      if (VAR != 2 && VAR != 3 && VAR < 5 && i < n) idx[dst] = (uint32_t)i;
      if (VAR == 2 && dst == 0xFFFFFFFFu) idx[0] = 1;
    }
    mbar_arrive(empty + k % kSStages);
  };
  if (tid == 0)
    for (int k = 0; k < kSLead && k < nst; ++k) produce(k);
  uint32_t d0 = 0, d1 = 0, d2 = 0;
  // step k: produce k+lead, claim k, store k-2 (slots rotate through d0, d1, d2)
  auto step = [&](int k, uint32_t& dk, uint32_t dold) {
    if (tid == 0 && k + kSLead < nst) produce(k + kSLead);
    if (k < nst) dk = claim(k);
    if (k >= kSDepth && k - kSDepth < nst) store(k - kSDepth, dold);
  };
  for (int k = 0; k < nst + kSDepth; k += 3) {  // unrolled by three: static slot registers
    step(k, d0, d1);
    step(k + 1, d1, d2);
    step(k + 2, d2, d0);
  }
}


int main() {
  const int64_t n = 1 << 24, m = 1 << 24, tot = n + m;
  const int L = 7;
  std::vector<double> h(3 * tot), hq(n);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  for (auto& v : h) v = U(rng);
  for (auto& v : hq) v = U(rng);
  double *pts, *q, *rec; uint32_t *cursor, *idx;
  cudaMalloc(&pts, 8 * 3 * tot); cudaMalloc(&q, 8 * n); cudaMalloc(&rec, 32 * tot + 64 * 1024 * 1024);
  cudaMalloc(&idx, 4 * tot + 4096); cudaMalloc(&cursor, 4 * 32 * 32768);
  cudaMemcpy(pts, h.data(), 8 * 3 * tot, cudaMemcpyHostToDevice);
  cudaMemcpy(q, hq.data(), 8 * n, cudaMemcpyHostToDevice);
  for (int bb : {14}) {
  BucketGeo g = bucket_geo(L, n, m, 148);
  g.bb = bb; g.shift = g.sbits - bb; g.nb = 2 << bb;
  // cursors: bucket b starts at b * cap (room for the bucket), like the real scan
  std::vector<uint32_t> hc(32 * 32768, 0);
  const uint32_t cap = (uint32_t)(tot / g.nb + tot / g.nb / 16 + 64);
  for (int b = 0; b < g.nb; ++b) hc[(size_t)b * 32] = (uint32_t)b * cap;
  printf("bb %d: %d buckets\n", bb, g.nb);
  int grid = 148;
  int64_t rows = scatter_rows_per_cta(tot, grid);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scatter_smem_bytes());
    float best = 1e9;
    for (int r = 0; r < 4; ++r) {
      cudaMemcpy(cursor, hc.data(), 4 * hc.size(), cudaMemcpyHostToDevice);
      cudaEventRecord(e0);
      kern<<<grid, kSThreads, scatter_smem_bytes()>>>(pts, q, pts + 3 * n, g, L, rows, cursor, rec, idx);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) best = ms < best ? ms : best;
    }
    printf("%-32s %8.1f us  %s\n", name, best * 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  run("full", k_var<true, 0>);
  run("no atomics (dst = i)", k_var<true, 1>);
  run("no stores", k_var<true, 2>);
  run("no idx store", k_var<true, 3>);
  run("8B store only (no idx)", k_var<true, 5>);
  run("2x16B store (no idx)", k_var<true, 6>);
  run("st.cs (no idx)", k_var<true, 7>);
  run("st.L1::no_allocate (no idx)", k_var<true, 8>);
  run("st.L2 evict_last (no idx)", k_var<true, 9>);
  }
}
