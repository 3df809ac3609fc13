// fif_cluster.cu -- host side of the cluster-resident regime (fif_cluster.cuh): geometry, tables, the
// per-cluster L2 scratch, and the cluster launch (cudaLaunchKernelEx with a cluster dimension).
#include <math.h>

#include <vector>

#include "fif_cluster.cuh"
#include "fif_plan.h"

namespace fifhost {
using namespace fifgpu;

namespace {
constexpr int kQ64 = 4096;  // fp64: 512 threads x 8 values per CTA

template <int P, int CAP>
using K64 = cl::Clu<double, kQ64, P, CAP>;

template <int P, int CAP>
void* kern64() {
  return (void*)cl::fif_cluster_kernel<double, kQ64, P, CAP>;
}
void* pick(int P, bool fast) {
  switch (P) {
    case 2: return fast ? kern64<2, kFastCap>() : kern64<2, 0>();
    case 4: return fast ? kern64<4, kFastCap>() : kern64<4, 0>();
    default: return fast ? kern64<8, kFastCap>() : kern64<8, 0>();
  }
}
size_t smem_of(int P) {
  switch (P) {
    case 2: return K64<2, 0>::smem_bytes;
    case 4: return K64<4, 0>::smem_bytes;
    default: return K64<8, 0>::smem_bytes;
  }
}
}  // namespace

// cluster size for a plan, 0 if the cluster regime does not cover it (fp64, n/2 = P 4096, P in {2, 4, 8})
int cl_cluster_size(int64_t n, fif_dtype dt) {
  if (dt != FIF_F64 || n % 2) return 0;
  const int64_t NC = n / 2;
  if (NC % kQ64) return 0;
  const int64_t P = NC / kQ64;
  return (P == 2 || P == 4 || P == 8) ? (int)P : 0;
}

fif_status cl_setup(fif_plan_s* p) {
  const int P = cl_cluster_size(p->n, p->dtype);
  if (!P) return FIF_ERR_UNSUPPORTED_N;
  p->cl_P = P;
  const int64_t n = p->n, NC = n / 2;
  // e^{i pi j / n}, j < 2n, two levels (the kernel's E()): Eh[h] = e^{i pi (h 2^9)/n}, El[l] = e^{i pi l/n}
  const int EB = 9, NEL = 1 << EB, NEH = (int)((2 * n) >> EB);
  const long double PI = 3.141592653589793238462643383279502884L;
  std::vector<double2> Eh(NEH), El(NEL);
  auto cis = [&](int64_t j) {
    const long double th = PI * (long double)j / (long double)n;
    return double2{(double)cosl(th), (double)sinl(th)};
  };
  for (int h = 0; h < NEH; ++h) Eh[h] = cis((int64_t)h << EB);
  for (int l = 0; l < NEL; ++l) El[l] = cis(l);
  // the local Q-point Stockham twiddles (the resident FFT's table for NC = Q)
  std::vector<double> sint, isin;
  std::vector<double2> tw;
  build_tables<double>(2 * kQ64, kQ64, sint, isin, tw);
  if (cudaMalloc(&p->d_Eh, sizeof(double2) * NEH) != cudaSuccess ||
      cudaMalloc(&p->d_El, sizeof(double2) * NEL) != cudaSuccess ||
      cudaMalloc(&p->d_tw, sizeof(double2) * tw.size()) != cudaSuccess)
    return FIF_ERR_OOM;
  if (cudaMemcpy(p->d_Eh, Eh.data(), sizeof(double2) * NEH, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->d_El, El.data(), sizeof(double2) * NEL, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->d_tw, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return FIF_ERR_CUDA;
  const size_t smem = smem_of(P);
  cudaError_t e = cudaSuccess;
  for (int fast = 0; fast < 2 && e == cudaSuccess; ++fast)
    e = cudaFuncSetAttribute(pick(P, fast), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    fprintf(stderr, "fif: cluster setup failed: %s\n", cudaGetErrorString(e));
    return FIF_ERR_CUDA;
  }
  // how many clusters fit at once (one CTA per SM; a cluster must fit in one GPC)
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(P * 64), 1, 1);
  cfg.blockDim = dim3(kQ64 / kR, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclu = 0;
  e = cudaOccupancyMaxActiveClusters(&nclu, pick(P, true), &cfg);
  if (e != cudaSuccess || nclu < 1) {
    fprintf(stderr, "fif: no cluster of %d CTAs fits (%s)\n", P, cudaGetErrorString(e));
    cudaGetLastError();
    return FIF_ERR_UNSUPPORTED_N;
  }
  p->cl_clusters = nclu;
  // per-cluster scratch: the mirror-publish and transpose regions (2 NC complex per cluster, L2-resident)
  const size_t per = (size_t)NC * sizeof(double2);
  if (cudaMalloc(&p->d_cl_scr, 2 * per * (size_t)nclu) != cudaSuccess) return FIF_ERR_OOM;
  p->block = kQ64 / kR;
  p->smem = smem;
  p->occ = 1;
  return FIF_OK;
}

void cl_decompose(fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its, int64_t batch,
                  cudaStream_t s) {
  if (batch <= 0) return;
  const int P = p->cl_P;
  int64_t G = p->cl_clusters;
  if (p->grid_cap > 0 && p->grid_cap / P >= 1 && p->grid_cap / P < G) G = p->grid_cap / P;
  if (batch < G) G = batch;
  Params prm{batch, p->xi, p->delta * p->delta, p->max_inner, p->max_imfs, (int32_t)p->window, p->stop,
             p->delta, p->gamma, p->mask};
  const size_t per = (size_t)p->n / 2 * sizeof(double2);
  cl::Scratch scr{p->d_cl_scr, (char*)p->d_cl_scr + per * (size_t)p->cl_clusters};
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(G * P), 1, 1);
  cfg.blockDim = dim3(kQ64 / kR, 1, 1);
  cfg.dynamicSmemBytes = p->smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const double* sg = (const double*)sig;
  double* out = (double*)imfs;
  const double2* Eh = (const double2*)p->d_Eh;
  const double2* El = (const double2*)p->d_El;
  const double2* tw = (const double2*)p->d_tw;
  const bool fast = p->max_inner == kFastCap;
  auto go = [&](auto kern) { cudaLaunchKernelEx(&cfg, kern, sg, out, cnt, lens, its, Eh, El, tw, scr, prm); };
  switch (P) {
    case 2:
      if (fast) go(cl::fif_cluster_kernel<double, kQ64, 2, kFastCap>); else go(cl::fif_cluster_kernel<double, kQ64, 2, 0>);
      break;
    case 4:
      if (fast) go(cl::fif_cluster_kernel<double, kQ64, 4, kFastCap>); else go(cl::fif_cluster_kernel<double, kQ64, 4, 0>);
      break;
    default:
      if (fast) go(cl::fif_cluster_kernel<double, kQ64, 8, kFastCap>); else go(cl::fif_cluster_kernel<double, kQ64, 8, 0>);
      break;
  }
}

void cl_free(fif_plan_s* p) { cudaFree(p->d_cl_scr); }
}  // namespace fifhost
