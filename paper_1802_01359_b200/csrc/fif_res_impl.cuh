// fif_res_impl.cuh -- resident-regime launchers for one element type (included by fif_res_f64.cu
// and fif_res_f32.cu, which compile in parallel).  Kernels: fif_resident.cuh.
#pragma once
#include "fif_plan.h"

namespace fifhost {
using namespace fifgpu;

template <typename Real, int NC>
struct Inst {
  using K = Resident<Real, NC>;
  using KT = Resident<Real, NC, 0, true>;  // table-driven instances (smaller shared-memory footprint)
  using V = typename Cx<Real>::V;
  // dynamic smem limit + a carveout just large enough for the occupancy the registers allow, so the rest
  // of the SM's 256 KB stays L1 (twiddles, table rows, spills)
  template <typename Kern>
  static cudaError_t main_attr(Kern k, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, K::T, smem)) != cudaSuccess) return e;
    const size_t need = (size_t)(occ > 0 ? occ : 1) * (smem + 1024);
    const int pct = (int)((need * 100 + 228 * 1024 - 1) / (228 * 1024));
    return cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
  }
  static cudaError_t prepare() {
    cudaError_t e;
    if ((e = main_attr(fif_resident_kernel<Real, NC, 0, false>, K::smem_bytes)) != cudaSuccess) return e;
    if ((e = main_attr(fif_resident_kernel<Real, NC, kFastCap, false>, K::smem_bytes)) != cudaSuccess) return e;
    if ((e = main_attr(fif_resident_kernel<Real, NC, 0, true>, KT::smem_bytes)) != cudaSuccess) return e;
    if ((e = main_attr(fif_resident_kernel<Real, NC, kFastCap, true>, KT::smem_bytes)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(fif_test_inner_kernel<Real, NC, kFastCap>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::smem_bytes)) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(fif_test_rfft_kernel<Real, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)K::smem_bytes)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(fif_test_irfft_kernel<Real, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)K::smem_bytes)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(fif_test_extrema_kernel<Real, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)K::smem_bytes)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(fif_test_window_kernel<Real, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)K::smem_bytes)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(fif_test_inner_kernel<Real, NC, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)K::smem_bytes)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(fif_wtab_kernel<Real, NC, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)K::smem_bytes)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(fif_wtab_kernel<Real, NC, kFastCap>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)K::smem_bytes)) != cudaSuccess) return e;
    return cudaSuccess;
  }
  static int occ_tab() {  // the table-mode instance's occupancy (its own register budget)
    static int occ = [] {
      int o = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fif_resident_kernel<Real, NC, kFastCap, true>, K::T,
                                                    KT::smem_bytes);
      return o > 0 ? o : 1;
    }();
    return occ;
  }
  static int occupancy() {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fif_resident_kernel<Real, NC, kFastCap, false>, K::T, K::smem_bytes);
    return occ;
  }
  static void decompose(const fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its,
                        int64_t batch, cudaStream_t s) {
    Params prm{batch, p->xi, p->delta * p->delta, p->max_inner, p->max_imfs, (int32_t)p->window, p->stop, p->delta, p->gamma, p->mask};
    prm.wtab = p->d_wtab;
    const bool fast = p->max_inner == kFastCap, tab = p->d_wtab != nullptr;
    auto kern = fast ? (tab ? fif_resident_kernel<Real, NC, kFastCap, true> : fif_resident_kernel<Real, NC, kFastCap, false>)
                     : (tab ? fif_resident_kernel<Real, NC, 0, true> : fif_resident_kernel<Real, NC, 0, false>);
    int64_t cap = (int64_t)p->num_sms * (tab ? occ_tab() : p->occ);  // persistent grid: one wave
    if (p->grid_cap > 0 && p->grid_cap < cap) cap = p->grid_cap;
    const int grid = (int)(batch < cap ? batch : cap);
    kern<<<grid, K::T, tab ? KT::smem_bytes : K::smem_bytes, s>>>((const Real*)sig, (Real*)imfs, cnt, lens, its,
                                                                 (const Real*)p->d_sin, (const Real*)p->d_isin,
                                                                 (const V*)p->d_tw, prm);
  }
  static void test_rfft(const fif_plan_s* p, const void* in, void* out, int64_t batch, cudaStream_t s) {
    const int grid = (int)(batch < 4096 ? batch : 4096);
    fif_test_rfft_kernel<Real, NC><<<grid, K::T, K::smem_bytes, s>>>(
        (const Real*)in, (Real*)out, batch, (const Real*)p->d_sin, (const Real*)p->d_isin, (const V*)p->d_tw);
  }
  static void test_irfft(const fif_plan_s* p, const void* in, void* out, int64_t batch, cudaStream_t s) {
    const int grid = (int)(batch < 4096 ? batch : 4096);
    fif_test_irfft_kernel<Real, NC><<<grid, K::T, K::smem_bytes, s>>>(
        (const Real*)in, (Real*)out, batch, (const Real*)p->d_sin, (const Real*)p->d_isin, (const V*)p->d_tw);
  }
  static void test_extrema(const fif_plan_s* p, const void* in, int32_t* k, int64_t batch, cudaStream_t s) {
    (void)p;
    const int grid = (int)(batch < 4096 ? batch : 4096);
    fif_test_extrema_kernel<Real, NC><<<grid, K::T, K::smem_bytes, s>>>((const Real*)in, k, batch);
  }
  static void test_window(const fif_plan_s* p, int L, void* out, cudaStream_t s) {
    fif_test_window_kernel<Real, NC><<<1, K::T, K::smem_bytes, s>>>((Real*)out, L, (const Real*)p->d_sin,
                                                                        (const Real*)p->d_isin);
  }
  static void fill_wtab(const fif_plan_s* p, void* tab, int nL, cudaStream_t s) {
    if (p->max_inner == kFastCap)
      fif_wtab_kernel<Real, NC, kFastCap><<<nL, K::T, K::smem_bytes, s>>>(tab, (const Real*)p->d_sin,
                                                                         (const Real*)p->d_isin, p->max_inner);
    else
      fif_wtab_kernel<Real, NC, 0><<<nL, K::T, K::smem_bytes, s>>>(tab, (const Real*)p->d_sin, (const Real*)p->d_isin,
                                                                  p->max_inner);
  }
  static void test_inner(const fif_plan_s* p, int L, const void* in, void* out, int32_t* N, int64_t batch,
                         cudaStream_t s) {
    Params prm{batch, p->xi, p->delta * p->delta, p->max_inner, p->max_imfs, (int32_t)p->window, p->stop, p->delta, p->gamma, p->mask};
    const int grid = (int)(batch < 4096 ? batch : 4096);
    if (p->max_inner == kFastCap)
      fif_test_inner_kernel<Real, NC, kFastCap><<<grid, K::T, K::smem_bytes, s>>>(
          (const Real*)in, (Real*)out, N, batch, L, (const Real*)p->d_sin, (const Real*)p->d_isin,
          (const V*)p->d_tw, prm);
    else
      fif_test_inner_kernel<Real, NC, 0><<<grid, K::T, K::smem_bytes, s>>>(
          (const Real*)in, (Real*)out, N, batch, L, (const Real*)p->d_sin, (const Real*)p->d_isin,
          (const V*)p->d_tw, prm);
  }
};


template <typename Real, int NC>
const ResOps* res_entry() {
  using I = Inst<Real, NC>;
  static const ResOps ops{&I::prepare,    &I::occupancy,  I::K::T,        I::K::smem_bytes, &I::decompose, &I::test_rfft,
                          &I::test_irfft, &I::test_extrema, &I::test_window, &I::test_inner, &I::fill_wtab};
  return &ops;
}
template <typename Real>
const ResOps* res_table(int NC) {
  switch (NC) {
    case 256: return res_entry<Real, 256>();
    case 512: return res_entry<Real, 512>();
    case 1024: return res_entry<Real, 1024>();
    case 2048: return res_entry<Real, 2048>();
    case 4096: return res_entry<Real, 4096>();
    case 8192:  // fp32 only: 1024 threads, 192 KB of shared memory (n = 16384, config 4)
      if constexpr (sizeof(Real) == 4) return res_entry<Real, 8192>();
      else return nullptr;
    default: return nullptr;
  }
}
}  // namespace fifhost
