// fif_plan.h -- internal: the plan object shared by the translation units of libfif_b200.so
// (fif.cu: C ABI; fif_res_f64.cu / fif_res_f32.cu: resident-regime launchers; fif_st.cu: streamed
// regime host code).  Not part of the public ABI (include/fif.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <math.h>
#include <nvtx3/nvToolsExt.h>

#include <vector>

#include "../../include/fif.h"
#include "fif_streamed.cuh"

namespace fifhost {
struct DistPlan;

// NVTX range for the duration of a scope (header-only NVTX3: a no-op unless a profiler such as nsys or
// ncu --nvtx is attached).  Names the host phases that enqueue the kernels of each regime.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

enum { FIF_MAX_STAGES = 3 };
// max_inner value with a compile-time-specialised kernel (the paper's/BASELINE's cap of 200,
// PAPER.md:433 "limit on the maximal number of iterations"); any other value uses the generic kernel
constexpr int kFastCap = 200;

struct Staging {
  void* d_in = nullptr;
  void* d_out = nullptr;
  int32_t* d_meta = nullptr;  // count | lens | iters
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
};

}  // namespace fifhost

struct fif_plan_s {
  int64_t n = 0, batch = 0;
  fif_dtype dtype = FIF_F64;
  fif_window window = FIF_WINDOW_TRI_SQ;
  double xi = 1.6, delta = 1e-3;
  int32_t max_inner = 200, max_imfs = 10;
  int32_t stop = 0;     // fif_stop_rule
  double gamma = 0.0;   // gamma-threshold (0: off)
  int32_t mask = 0;     // fif_mask_rule
  int device = 0, num_sms = 0;
  int NC = 0;
  void* d_sin = nullptr;   // Real[NC+1]  sin(pi j/n)
  void* d_isin = nullptr;  // Real[NC+1]  1/sin(pi j/n) (j >= 1)
  void* d_tw = nullptr;    // V[twtotal]  Stockham twiddles e^{-2 pi i k r/(NS RP)}
  void* d_wtab = nullptr;  // Real[(n-1)/4 - 1][NC+1][2] per-L eigenvalue table (fif_plan_set_eigen_table)
  int block = 0, occ = 0;
  int grid_cap = 0;        // > 0: persistent grids capped at this many CTAs (FIF_GRID_CAP at creation; tests)
  size_t smem = 0;
  int regime = 0;  // 0 resident, 1 streamed, 2 distributed, 3 iterative, 4 cluster
  // cluster regime (fif_cluster.cu)
  int cl_P = 0, cl_clusters = 0;
  void* d_cl_scr = nullptr;  // per-cluster L2 scratch (mirror publish + transpose landing regions)
  // streamed regime
  fifgpu::st::Geo geo{};
  void* d_Eh = nullptr;   // double2 e^{i pi (h 2^eb)/n}
  void* d_El = nullptr;   // double2 e^{i pi l/n}
  void* d_Th = nullptr;   // V (Real) copies
  void* d_Tl = nullptr;
  void* d_twl = nullptr;  // V per-level Stockham twiddles
  // decompose workspace (fif_plan_workspace_bytes): d_X | d_Xn | d_ctl [| d_pnat], carved from one block --
  // plan-owned (d_ws_own) unless the caller handed its own (fif_plan_set_workspace, d_ws_user)
  void* d_ws_own = nullptr;
  void* d_ws_user = nullptr;
  size_t ws_user_bytes = 0;
  size_t ws_xn = 0, ws_ctl = 0, ws_pnat = 0, ws_end = 0, ws_end_pnat = 0;  // offsets (bytes)
  size_t ws_ctl_bytes = 0;
  void* d_X = nullptr;    // V[2][B][NC] spectrum ping-pong (digit-reversed multi-level order)
  void* d_Xn = nullptr;   // V[2][B] Nyquist bins
  void* d_ctl = nullptr;  // per-signal control arrays + partials
  void* d_utab = nullptr;   // int2[units] mirror-pair rows
  void* d_pnat = nullptr;   // double[B][NC+1] natural-order powers (spectral-peak rule only; in the workspace)
  void* d_rbase = nullptr;  // int[rows] row bin bases
  void* d_rmir = nullptr;   // int[rows] mirror rows
  fifgpu::st::Ctl ctl{};
  int st_rounds = 0, st_grid = 0, st_grid_col = 0, st_grid_rows = 0, st_grid_probe = 0;
  int64_t st_wave = 1;
  fifhost::DistPlan* dist = nullptr;  // distributed regime (fif_dist.cu)
  cudaStream_t st_streams[2] = {nullptr, nullptr};  // waves alternate between these
  cudaEvent_t st_ev[3] = {nullptr, nullptr, nullptr};
  size_t st_smem_col[fifgpu::st::kMaxLev] = {}, st_smem_rows = 0, st_smem_rows_inv = 0;
  int st_col_cs[fifgpu::st::kMaxLev] = {};  // column transform path per level (st::col_fft CS)
  int st_col_rm[fifgpu::st::kMaxLev] = {};  // the same with row-major bulk-copy-staged tiles (CS + 20), 0: unavailable
  int st_col_tm[fifgpu::st::kMaxLev] = {};  // 1: the row-major tile is one cp.async.bulk.tensor box (tensor map per call)
  int st_row_rs = 0;                         // row transform path (st::row_fft RS)
  // host (e2e) path staging
  int64_t chunk = 0;
  int nstages = 0;
  fifhost::Staging st[fifhost::FIF_MAX_STAGES];
};

namespace fifhost {
using fifgpu::Cx;
// ---------------------------------------------------------------- tables (host, long double)
// sin(pi j/n), 1/sin(pi j/n) (j <= NC) and the Stockham twiddles of the resident FFT of NC points
template <typename Real>
inline void build_tables(int64_t n, int NC, std::vector<Real>& sint, std::vector<Real>& isin,
                  std::vector<typename Cx<Real>::V>& tw) {
  const long double PI = 3.141592653589793238462643383279502884L;
  sint.assign(NC + 1, (Real)0);
  isin.assign(NC + 1, (Real)0);
  for (int j = 0; j <= NC; ++j) {
    // sin(pi j / n), j <= n/2; reflect to keep the argument <= pi/4 for accuracy
    long double v;
    if (2 * (int64_t)j <= n / 2) v = sinl(PI * (long double)j / (long double)n);
    else v = cosl(PI * (long double)(n / 2 - j) / (long double)n);
    sint[j] = (Real)v;
    isin[j] = j ? (Real)(1.0L / v) : (Real)0;
  }
  const int P = fifgpu::sched_passes(NC);
  tw.assign(fifgpu::sched_twtotal(NC) > 0 ? fifgpu::sched_twtotal(NC) : 1, typename Cx<Real>::V{0, 0});
  for (int p = 1; p < P; ++p) {
    const int RP = fifgpu::sched_radix(NC, p), NS = fifgpu::sched_ns(NC, p), off = fifgpu::sched_twoff(NC, p);
    const int64_t den = (int64_t)NS * RP;
    for (int r = 1; r < RP; ++r)
      for (int k = 0; k < NS; ++k) {
        const int64_t m = ((int64_t)k * r) % den;
        const long double th = 2.0L * PI * (long double)m / (long double)den;
        tw[off + (r - 1) * NS + k] = typename Cx<Real>::V{(Real)cosl(th), (Real)(-sinl(th))};
      }
  }
}

// resident regime: per-(dtype, NC) launchers (fif_res_f64.cu, fif_res_f32.cu)
struct ResOps {
  cudaError_t (*prepare)();
  int (*occupancy)();
  int threads;
  size_t smem;
  void (*decompose)(const fif_plan_s*, const void*, void*, int32_t*, int32_t*, int32_t*, int64_t, cudaStream_t);
  void (*test_rfft)(const fif_plan_s*, const void*, void*, int64_t, cudaStream_t);
  void (*test_irfft)(const fif_plan_s*, const void*, void*, int64_t, cudaStream_t);
  void (*test_extrema)(const fif_plan_s*, const void*, int32_t*, int64_t, cudaStream_t);
  void (*test_window)(const fif_plan_s*, int, void*, cudaStream_t);
  void (*test_inner)(const fif_plan_s*, int, const void*, void*, int32_t*, int64_t, cudaStream_t);
  void (*fill_wtab)(const fif_plan_s*, void*, int, cudaStream_t);
};
const ResOps* res_ops_f64(int NC);
const ResOps* res_ops_f32(int NC);
inline const ResOps* res_ops(fif_dtype dt, int NC) { return dt == FIF_F64 ? res_ops_f64(NC) : res_ops_f32(NC); }

// streamed regime (fif_st.cu)
bool st_geometry(int64_t n, bool f64, fifgpu::st::Geo& g);
fif_status st_row_tables(const fifgpu::st::Geo& g, void** d_utab, void** d_rbase, void** d_rmir);
fif_status st_setup(fif_plan_s* p);
// signals [0, batch) of the call use the plan's work buffers from signal `boff` on
void st_decompose(fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its,
                  int64_t batch, int64_t boff, cudaStream_t s);
int st_kernels_per_call(const fif_plan_s* p);
void st_free(fif_plan_s* p);
// workspace: bytes needed with the current options; (re)bind the buffers to `base` (nullptr: plan-owned block)
size_t st_workspace_bytes(const fif_plan_s* p);
fif_status st_bind_workspace(fif_plan_s* p, void* base, size_t bytes);
// compile-time transform path of a C x F tile level (st::col_fft CS; 0 = generic)
int pass_schedule(const fifgpu::st::Level& lv, bool f64);

// cluster-resident regime (fif_cluster.cu): one signal per thread-block cluster, r and r_hat on chip
int cl_cluster_size(int64_t n, fif_dtype dt);  // 0: not covered
fif_status cl_setup(fif_plan_s* p);
void cl_decompose(fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its, int64_t batch,
                  cudaStream_t s);
void cl_free(fif_plan_s* p);

// iterative regime (fif_iterative.cu): Algorithm 2 literally (the IF baseline of PAPER.md:693)
fif_status it_setup(fif_plan_s* p);
void it_decompose(fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its, int64_t batch,
                  cudaStream_t s);

// distributed regime (fif_dist.cu): one signal time-block sharded over nranks GPUs
fif_status dist_create(fif_plan_s* p, const void* nccl_uid, int rank, int nranks, int emulated);
fif_status dist_decompose(fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its,
                          cudaStream_t s);
void dist_free(fif_plan_s* p);
int dist_kernels_per_call(const fif_plan_s* p);
fif_status nccl_unique_id(void* out);
}  // namespace fifhost
