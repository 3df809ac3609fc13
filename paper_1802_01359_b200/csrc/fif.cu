// fif.cu -- C ABI of the B200 FIF hot path (include/fif.h): plan creation
// (validation, device tables), dispatch to the sm_100a kernels, the host-buffer
// end-to-end path and the test hooks.  No torch types, no CPU compute fallback:
// every step of the decomposition runs in the kernels of fif_resident.cuh.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <utility>

#include <vector>

#include "../../include/fif.h"
#include "fif_resident.cuh"
#include "fif_streamed.cuh"

using namespace fifgpu;

namespace {

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

}  // namespace

struct fif_plan_s {
  int64_t n = 0, batch = 0;
  fif_dtype dtype = FIF_F64;
  fif_window window = FIF_WINDOW_TRI_SQ;
  double xi = 1.6, delta = 1e-3;
  int32_t max_inner = 200, max_imfs = 10;
  int device = 0, num_sms = 0;
  int NC = 0;
  void* d_sin = nullptr;   // Real[NC+1]  sin(pi j/n)
  void* d_isin = nullptr;  // Real[NC+1]  1/sin(pi j/n) (j >= 1)
  void* d_tw = nullptr;    // V[twtotal]  Stockham twiddles e^{-2 pi i k r/(NS RP)}
  int block = 0, occ = 0;
  size_t smem = 0;
  int regime = 0;  // 0 resident, 1 streamed
  // streamed regime
  st::Geo geo{};
  void* d_Eh = nullptr;   // double2 e^{i pi (h 2^eb)/n}
  void* d_El = nullptr;   // double2 e^{i pi l/n}
  void* d_Th = nullptr;   // V (Real) copies
  void* d_Tl = nullptr;
  void* d_twl = nullptr;  // V per-level Stockham twiddles
  void* d_X = nullptr;    // V[B][NC] spectrum (digit-reversed multi-level order)
  void* d_Xn = nullptr;   // V[B] Nyquist bins
  void* d_ctl = nullptr;  // per-signal control arrays + partials
  st::Ctl ctl{};
  int st_rounds = 0, st_grid = 0, st_grid_col = 0, st_grid_rows = 0, st_grid_probe = 0;
  int64_t st_wave = 1;
  size_t st_smem_col[st::kMaxLev] = {}, st_smem_rows = 0;
  // host (e2e) path staging
  int64_t chunk = 0;
  int nstages = 0;
  Staging st[FIF_MAX_STAGES];
};

namespace {


// ---------------------------------------------------------------- kernel table
struct Entry {
  int NC;
  int R;
  size_t smem;
  int threads;
};

template <typename Real, int NC>
struct Inst {
  using K = Resident<Real, NC>;
  using V = typename Cx<Real>::V;
  static cudaError_t prepare() {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(fif_resident_kernel<Real, NC, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)K::smem_bytes)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(fif_resident_kernel<Real, NC, kFastCap>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)K::smem_bytes)) != cudaSuccess) return e;
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
    return cudaSuccess;
  }
  static int occupancy() {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fif_resident_kernel<Real, NC, kFastCap>, K::T, K::smem_bytes);
    return occ;
  }
  static void decompose(const fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its,
                        int64_t batch, cudaStream_t s) {
    Params prm{batch, p->xi, p->delta * p->delta, p->max_inner, p->max_imfs, (int32_t)p->window};
    const int64_t cap = (int64_t)p->num_sms * p->occ;
    const int grid = (int)(batch < cap ? batch : cap);
    if (p->max_inner == kFastCap)
      fif_resident_kernel<Real, NC, kFastCap><<<grid, K::T, K::smem_bytes, s>>>(
          (const Real*)sig, (Real*)imfs, cnt, lens, its, (const Real*)p->d_sin, (const Real*)p->d_isin,
          (const V*)p->d_tw, prm);
    else
      fif_resident_kernel<Real, NC, 0><<<grid, K::T, K::smem_bytes, s>>>(
          (const Real*)sig, (Real*)imfs, cnt, lens, its, (const Real*)p->d_sin, (const Real*)p->d_isin,
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
  static void test_inner(const fif_plan_s* p, int L, const void* in, void* out, int32_t* N, int64_t batch,
                         cudaStream_t s) {
    Params prm{batch, p->xi, p->delta * p->delta, p->max_inner, p->max_imfs, (int32_t)p->window};
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

// Dispatch on (dtype, NC).  F is a functor template taking Inst<Real,NC,R>.
template <typename Real, typename F>
bool dispatch_nc(int NC, F&& f) {
  switch (NC) {
    case 256: f(Inst<Real, 256>{}); return true;
    case 512: f(Inst<Real, 512>{}); return true;
    case 1024: f(Inst<Real, 1024>{}); return true;
    case 2048: f(Inst<Real, 2048>{}); return true;
    case 4096: f(Inst<Real, 4096>{}); return true;
    default: return false;
  }
}
template <typename F>
bool dispatch(fif_dtype dt, int NC, F&& f) {
  if (dt == FIF_F64) return dispatch_nc<double>(NC, f);
  return dispatch_nc<float>(NC, f);
}

// ---------------------------------------------------------------- tables (host, long double)
template <typename Real>
void build_tables(int64_t n, int NC, std::vector<Real>& sint, std::vector<Real>& isin,
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
  const int P = sched_passes(NC);
  tw.assign(sched_twtotal(NC) > 0 ? sched_twtotal(NC) : 1, typename Cx<Real>::V{0, 0});
  for (int p = 1; p < P; ++p) {
    const int RP = sched_radix(NC, p), NS = sched_ns(NC, p), off = sched_twoff(NC, p);
    const int64_t den = (int64_t)NS * RP;
    for (int r = 1; r < RP; ++r)
      for (int k = 0; k < NS; ++k) {
        const int64_t m = ((int64_t)k * r) % den;
        const long double th = 2.0L * PI * (long double)m / (long double)den;
        tw[off + (r - 1) * NS + k] = typename Cx<Real>::V{(Real)cosl(th), (Real)(-sinl(th))};
      }
  }
}

template <typename Real>
fif_status upload_tables(fif_plan_s* p) {
  std::vector<Real> sint, isin;
  std::vector<typename Cx<Real>::V> tw;
  build_tables<Real>(p->n, p->NC, sint, isin, tw);
  if (cudaMalloc(&p->d_sin, sizeof(Real) * sint.size()) != cudaSuccess) return FIF_ERR_OOM;
  if (cudaMalloc(&p->d_isin, sizeof(Real) * isin.size()) != cudaSuccess) return FIF_ERR_OOM;
  if (cudaMalloc(&p->d_tw, sizeof(tw[0]) * tw.size()) != cudaSuccess) return FIF_ERR_OOM;
  if (cudaMemcpy(p->d_sin, sint.data(), sizeof(Real) * sint.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->d_isin, isin.data(), sizeof(Real) * isin.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->d_tw, tw.data(), sizeof(tw[0]) * tw.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return FIF_ERR_CUDA;
  return FIF_OK;
}

size_t elem_size(fif_dtype d) { return d == FIF_F64 ? 8 : 4; }

fif_status launch_status() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "fif: CUDA error: %s\n", cudaGetErrorString(e));
    return FIF_ERR_CUDA;
  }
  return FIF_OK;
}


// ---------------------------------------------------------------- streamed regime (fif_streamed.cuh)
bool smooth235(int64_t x) {
  if (x < 1) return false;
  for (int f : {2, 3, 5})
    while (x % f == 0) x /= f;
  return x == 1;
}
// radix schedule: 8s, then the leftover power of two (4 or 2), then 3s and 5s
int radices(int64_t N, int* rad) {
  int np = 0, a = 0;
  while (N % 2 == 0) { N /= 2; ++a; }
  while (a >= 3) { rad[np++] = 8; a -= 3; }
  if (a == 2) rad[np++] = 4;
  if (a == 1) rad[np++] = 2;
  while (N % 3 == 0) { N /= 3; rad[np++] = 3; }
  while (N % 5 == 0) { N /= 5; rad[np++] = 5; }
  return np;
}
// split x into m factors, each smooth and in [2, fmax], largest first
bool split_factors(int64_t x, int m, int64_t fmax, std::vector<int64_t>& out) {
  if (m == 1) {
    if (x >= 2 && x <= fmax && smooth235(x)) { out.push_back(x); return true; }
    return false;
  }
  for (int64_t d = fmax < x ? fmax : x; d >= 2; --d) {
    if (x % d || !smooth235(d)) continue;
    out.push_back(d);
    if (split_factors(x / d, m - 1, fmax, out)) return true;
    out.pop_back();
  }
  return false;
}
// Multi-level geometry: NC = F_0 ... F_{L-1}; the row level holds a mirror pair of rows (2 F_{L-1}
// complex values per smem buffer), the column levels F_i C_i values with C_i >= 128 B of columns.
bool st_geometry(int64_t n, bool f64, st::Geo& g) {
  const int64_t NC = n / 2;
  const int64_t Emax = f64 ? 2048 : 4096;
  int64_t rowmax = Emax / 2, colmax = Emax / (f64 ? 8 : 16);
  // test-only knobs: smaller level lengths force 3- and 4-level geometries at small n
  if (getenv("FIF_ST_ROWMAX")) rowmax = atoll(getenv("FIF_ST_ROWMAX"));
  if (getenv("FIF_ST_COLMAX")) colmax = atoll(getenv("FIF_ST_COLMAX"));
  if (n % 2 || NC < 4 || !smooth235(NC)) return false;
  for (int L = 2; L <= st::kMaxLev; ++L) {
    for (int64_t row = rowmax < NC / 2 ? rowmax : NC / 2; row >= 2; --row) {
      if (NC % row || !smooth235(row)) continue;
      std::vector<int64_t> f;
      if (!split_factors(NC / row, L - 1, colmax, f)) continue;
      // level 0 gets the smallest factor (widest tiles: long extrema segments, coalesced rows)
      std::vector<int64_t> F(f.rbegin(), f.rend());
      F.push_back(row);
      g = st::Geo{};
      g.n = n; g.NC = NC; g.L = L;
      int twoff = 0;
      for (int i = 0; i < L; ++i) {
        st::Level& lv = g.lv[i];
        lv.F = (int)F[i];
        int64_t S = 1;
        for (int j = i + 1; j < L; ++j) S *= F[j];
        lv.S = S;
        lv.A = NC / (F[i] * S);
        lv.E2 = 2 * n / (F[i] * S);
        lv.np = radices(F[i], lv.rad);
        lv.twoff = twoff;
        twoff += lv.F;
        if (i < L - 1) {
          int64_t cmax = Emax / F[i], C = 1;
          for (int64_t c = cmax < S ? cmax : S; c >= 1; --c)
            if (S % c == 0) { C = c; break; }
          lv.C = (int)C;
          lv.pitch = lv.F + 1;
          lv.tiles = lv.A * S / C;
        } else {
          lv.C = 2;
          lv.pitch = lv.F;
          lv.tiles = 0;
        }
        g.Fd[i] = lv.F;
        g.Pd[i] = i == 0 ? 1 : g.Pd[i - 1] * F[i - 1];
        g.Sr[i] = S / row;
      }
      g.Frow = (int)row;
      g.P = NC / row;
      g.units = g.P / 2 + 1;
      g.nseg = NC / g.lv[0].C;
      g.grp = 2048;
      g.ngrp = (g.nseg + g.grp - 1) / g.grp;
      g.rpc = 8192 / row > 1 ? 8192 / row : 1;
      g.nbch = (g.P + g.rpc - 1) / g.rpc;
      int bits = 0;
      while ((1LL << bits) < 2 * n + 1) ++bits;
      g.eb = (bits + 1) / 2;
      return true;
    }
  }
  return false;
}
template <typename Real>
fif_status st_tables(fif_plan_s* p) {
  using V = typename Cx<Real>::V;
  const long double PI = 3.141592653589793238462643383279502884L;
  const st::Geo& g = p->geo;
  const int64_t nh = (2 * g.n >> g.eb) + 1, nl = 1LL << g.eb;
  auto cis = [&](int64_t j) {  // e^{i pi j/n}, argument reduced to [0, pi/4] for accuracy
    const int64_t n = g.n, j2 = j % (2 * n);
    // angle pi j2/n; use symmetry: quadrant q = floor(2 j2 / n)
    long double c = cosl(PI * (long double)j2 / (long double)n), s = sinl(PI * (long double)j2 / (long double)n);
    return std::pair<long double, long double>(c, s);
  };
  std::vector<double2> Eh(nh), El(nl);
  std::vector<V> Th(nh), Tl(nl);
  for (int64_t h = 0; h < nh; ++h) {
    auto cs = cis(h << g.eb);
    Eh[h] = double2{(double)cs.first, (double)cs.second};
    Th[h] = V{(Real)cs.first, (Real)cs.second};
  }
  for (int64_t l = 0; l < nl; ++l) {
    auto cs = cis(l);
    El[l] = double2{(double)cs.first, (double)cs.second};
    Tl[l] = V{(Real)cs.first, (Real)cs.second};
  }
  std::vector<V> tw;
  for (int i = 0; i < g.L; ++i)
    for (int j = 0; j < g.lv[i].F; ++j) {
      const long double th = 2.0L * PI * (long double)j / (long double)g.lv[i].F;
      tw.push_back(V{(Real)cosl(th), (Real)(-sinl(th))});
    }
  auto up = [](void** d, const void* h, size_t bytes) {
    if (cudaMalloc(d, bytes) != cudaSuccess) return FIF_ERR_OOM;
    return cudaMemcpy(*d, h, bytes, cudaMemcpyHostToDevice) == cudaSuccess ? FIF_OK : FIF_ERR_CUDA;
  };
  fif_status s;
  if ((s = up(&p->d_Eh, Eh.data(), sizeof(double2) * nh)) != FIF_OK) return s;
  if ((s = up(&p->d_El, El.data(), sizeof(double2) * nl)) != FIF_OK) return s;
  if ((s = up(&p->d_Th, Th.data(), sizeof(V) * nh)) != FIF_OK) return s;
  if ((s = up(&p->d_Tl, Tl.data(), sizeof(V) * nl)) != FIF_OK) return s;
  if ((s = up(&p->d_twl, tw.data(), sizeof(V) * tw.size())) != FIF_OK) return s;
  return FIF_OK;
}
template <typename K>
int occ_grid(const fif_plan_s* p, K kern, size_t smem) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, st::kThreads, smem);
  return p->num_sms * (occ > 0 ? occ : 1);
}
template <typename Real>
fif_status st_setup(fif_plan_s* p) {
  using V = typename Cx<Real>::V;
  st::Geo& g = p->geo;
  if (!st_geometry(p->n, sizeof(Real) == 8, g)) return FIF_ERR_UNSUPPORTED_N;
  g.batch = p->batch;
  g.max_imfs = p->max_imfs; g.max_inner = p->max_inner; g.window = (int)p->window;
  g.xi = p->xi; g.delta2 = p->delta * p->delta;
  g.sig_stride = (int64_t)(p->max_imfs + 1) * p->n;
  p->st_rounds = 0;  // K-ary rounds: the bracket shrinks from cap to ceil(len / (kProbes + 1)) per round
  for (int64_t len = p->max_inner; len > 1; len = (len + st::kProbes) / (st::kProbes + 1)) ++p->st_rounds;
  fif_status s = st_tables<Real>(p);
  if (s != FIF_OK) return s;
  // L2 waves: the working set of a signal (spectrum, remainder, IMF slot: 3 n b bytes) of a wave
  // of signals stays in the 126 MB L2 across the passes of an IMF
  const double wave_mb = getenv("FIF_WAVE_MB") ? atof(getenv("FIF_WAVE_MB")) : 64.0;
  const int64_t per_sig = 3 * p->n * (int64_t)sizeof(Real);
  int64_t wave = (int64_t)(wave_mb * 1048576.0 / (double)per_sig);
  if (wave < 1) wave = 1;
  const int64_t B = p->batch > 0 ? p->batch : 1;
  if (wave > B) wave = B;
  p->st_wave = wave;
  const size_t ni = (size_t)B * 10;
  const size_t segb = (size_t)B * g.nseg * (sizeof(uint32_t) + 2 * sizeof(Real));
  const size_t grpb = (size_t)B * g.ngrp * (sizeof(uint32_t) + 2 * sizeof(Real));
  const size_t redb = (size_t)B * g.nbch * 2 * st::kProbes * sizeof(double);
  const size_t ctl_bytes = ni * sizeof(int32_t) + segb + grpb + redb + 256;
  if (cudaMalloc(&p->d_X, sizeof(V) * B * g.NC) != cudaSuccess || cudaMalloc(&p->d_Xn, sizeof(V) * B) != cudaSuccess ||
      cudaMalloc(&p->d_ctl, ctl_bytes) != cudaSuccess)
    return FIF_ERR_OOM;
  char* q = (char*)p->d_ctl;
  auto take = [&](size_t bytes) {
    char* r = q;
    q += (bytes + 15) & ~(size_t)15;
    return (void*)r;
  };
  st::Ctl& c = p->ctl;
  c.red = (double*)take(redb);
  c.segv = take((size_t)B * g.nseg * 2 * sizeof(Real));
  c.gv = take((size_t)B * g.ngrp * 2 * sizeof(Real));
  c.segi = (uint32_t*)take((size_t)B * g.nseg * sizeof(uint32_t));
  c.gi = (uint32_t*)take((size_t)B * g.ngrp * sizeof(uint32_t));
  int32_t* ip = (int32_t*)take(ni * sizeof(int32_t));
  c.k = ip; c.L = ip + B; c.N = ip + 2 * B; c.M = ip + 3 * B; c.active = ip + 4 * B; c.search = ip + 5 * B;
  c.lo = ip + 6 * B; c.hi = ip + 7 * B; c.bad = ip + 8 * B; c.cnt = (uint32_t*)(ip + 9 * B);
  if (cudaMemset(p->d_ctl, 0, ctl_bytes) != cudaSuccess) return FIF_ERR_CUDA;
  // shared memory and grids
  for (int i = 0; i < g.L - 1; ++i) p->st_smem_col[i] = 2 * sizeof(V) * (size_t)g.lv[i].C * g.lv[i].pitch;
  p->st_smem_rows = 2 * sizeof(V) * 2 * (size_t)g.lv[g.L - 1].pitch;
  size_t smax = p->st_smem_rows;
  for (int i = 0; i < g.L - 1; ++i) smax = smax > p->st_smem_col[i] ? smax : p->st_smem_col[i];
  cudaError_t e = cudaSuccess;
  auto attr = [&](auto kern) {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
  };
  attr(st::k_col<Real, -1, st::PASS_FWD_FIRST>);
  attr(st::k_col<Real, -1, st::PASS_MID>);
  attr(st::k_col<Real, 1, st::PASS_MID>);
  attr(st::k_col<Real, 1, st::PASS_INV_LAST>);
  attr(st::k_rows_fwd<Real>);
  attr(st::k_rows_inv<Real>);
  if (e != cudaSuccess) {
    fprintf(stderr, "fif: streamed setup failed: %s\n", cudaGetErrorString(e));
    return FIF_ERR_CUDA;
  }
  p->st_grid_col = occ_grid(p, st::k_col<Real, 1, st::PASS_INV_LAST>, smax);
  p->st_grid_rows = occ_grid(p, st::k_rows_inv<Real>, p->st_smem_rows);
  p->st_grid_probe = occ_grid(p, st::k_probe<Real>, 0);
  p->st_grid = p->st_grid_rows;
  p->block = st::kThreads;
  p->smem = smax;
  p->occ = 1;
  return FIF_OK;
}

// Ctl / geometry of the wave of signals [b0, b0 + nb)
st::Ctl ctl_at(const st::Ctl& c, const st::Geo& g, int64_t b0, size_t rsz) {
  st::Ctl r = c;
  r.k += b0; r.L += b0; r.N += b0; r.M += b0; r.active += b0; r.search += b0; r.lo += b0; r.hi += b0;
  r.bad += b0; r.cnt += b0;
  r.segi += b0 * g.nseg;
  r.segv = (char*)c.segv + b0 * g.nseg * 2 * rsz;
  r.gi += b0 * g.ngrp;
  r.gv = (char*)c.gv + b0 * g.ngrp * 2 * rsz;
  r.red += b0 * g.nbch * 2 * st::kProbes;
  return r;
}
int grid_for(int64_t work, int cap) { return (int)(work < cap ? (work > 0 ? work : 1) : cap); }

// the whole decomposition as stream-ordered kernels (no host synchronisation), one L2 wave at a time
template <typename Real>
void st_decompose(fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its, int64_t batch,
                  cudaStream_t s) {
  using V = typename Cx<Real>::V;
  const int TB = st::kThreads;
  const st::Tabs<Real> tb{(const double2*)p->d_Eh, (const double2*)p->d_El, (const V*)p->d_Th, (const V*)p->d_Tl,
                          (const V*)p->d_twl};
  for (int64_t b0 = 0; b0 < batch; b0 += p->st_wave) {
    st::Geo g = p->geo;
    g.batch = batch - b0 < p->st_wave ? batch - b0 : p->st_wave;
    const st::Ctl c = ctl_at(p->ctl, g, b0, sizeof(Real));
    const Real* sg = (const Real*)sig + b0 * g.n;
    Real* out = (Real*)imfs + b0 * g.sig_stride;
    V* X = (V*)p->d_X + b0 * g.NC;
    V* Xn = (V*)p->d_Xn + b0;
    int32_t* ln = lens + b0 * g.max_imfs;
    int32_t* it = its + b0 * g.max_imfs;
    const int Lv = g.L;
    const st::Level& top = g.lv[Lv - 1];
    const int gcol = p->st_grid_col, grow = grid_for(g.batch * g.units, p->st_grid_rows);
    const int gprobe = grid_for(g.batch * g.nbch, p->st_grid_probe);
    const int gfold = grid_for(g.batch * g.ngrp, p->num_sms * 4);
    const int gsig = (int)((g.batch + TB - 1) / TB);
    auto col = [&](int i) { return grid_for(g.batch * g.lv[i].tiles, gcol); };
    st::k_init<<<gsig, TB, 0, s>>>(g, c);
    st::k_col<Real, -1, st::PASS_FWD_FIRST><<<col(0), TB, p->st_smem_col[0], s>>>(g, g.lv[0], sg, out, X, tb, c);
    st::k_fold<Real><<<gfold, TB, 0, s>>>(g, c, 0, ln, it);
    for (int i = 1; i < Lv - 1; ++i)
      st::k_col<Real, -1, st::PASS_MID><<<col(i), TB, p->st_smem_col[i], s>>>(g, g.lv[i], sg, out, X, tb, c);
    st::k_rows_fwd<Real><<<grow, TB, p->st_smem_rows, s>>>(g, top, X, Xn, tb, c);
    for (int m = 0; m < g.max_imfs; ++m) {
      st::k_probe<Real><<<gprobe, TB, 0, s>>>(g, X, Xn, tb, c, 0);
      for (int r = 0; r < p->st_rounds; ++r) st::k_probe<Real><<<gprobe, TB, 0, s>>>(g, X, Xn, tb, c, 1);
      st::k_rows_inv<Real><<<grow, TB, p->st_smem_rows, s>>>(g, top, out, X, Xn, tb, c);
      for (int i = Lv - 2; i >= 1; --i)
        st::k_col<Real, 1, st::PASS_MID><<<col(i), TB, p->st_smem_col[i], s>>>(g, g.lv[i], sg, out, X, tb, c);
      st::k_col<Real, 1, st::PASS_INV_LAST><<<col(0), TB, p->st_smem_col[0], s>>>(g, g.lv[0], sg, out, X, tb, c);
      st::k_fold<Real><<<gfold, TB, 0, s>>>(g, c, 1, ln, it);
    }
    st::k_final<Real><<<grid_for(g.batch, p->num_sms * 4), TB, 0, s>>>(g, out, c, cnt + b0, ln, it);
  }
}
int st_kernels_per_call(const fif_plan_s* p) {
  const int L = p->geo.L;
  const int64_t waves = p->batch > 0 ? (p->batch + p->st_wave - 1) / p->st_wave : 0;
  return (int)(waves * (2 + (L - 1) + 1 + p->max_imfs * (1 + p->st_rounds + L + 1) + 1));
}

void free_plan(fif_plan_s* p) {
  if (!p) return;
  cudaFree(p->d_sin);
  cudaFree(p->d_isin);
  cudaFree(p->d_tw);
  cudaFree(p->d_Eh);
  cudaFree(p->d_El);
  cudaFree(p->d_Th);
  cudaFree(p->d_Tl);
  cudaFree(p->d_twl);
  cudaFree(p->d_X);
  cudaFree(p->d_Xn);
  cudaFree(p->d_ctl);
  for (int i = 0; i < p->nstages; ++i) {
    cudaFree(p->st[i].d_in);
    cudaFree(p->st[i].d_out);
    cudaFree(p->st[i].d_meta);
    if (p->st[i].stream) cudaStreamDestroy(p->st[i].stream);
    if (p->st[i].done) cudaEventDestroy(p->st[i].done);
  }
  delete p;
}

}  // namespace

extern "C" {

const char* fif_status_string(fif_status s) {
  switch (s) {
    case FIF_OK: return "FIF_OK";
    case FIF_ERR_INVALID_ARG: return "FIF_ERR_INVALID_ARG";
    case FIF_ERR_UNSUPPORTED_N: return "FIF_ERR_UNSUPPORTED_N";
    case FIF_ERR_OOM: return "FIF_ERR_OOM";
    case FIF_ERR_CUDA: return "FIF_ERR_CUDA";
    case FIF_ERR_NCCL: return "FIF_ERR_NCCL";
  }
  return "FIF_ERR_UNKNOWN";
}

fif_status fif_plan_create(fif_plan_t* out, int64_t n, int64_t batch, fif_dtype dtype, fif_window window, double xi,
                           double delta, int32_t max_inner, int32_t max_imfs) {
  return fif_plan_create_ex(out, n, batch, dtype, window, xi, delta, max_inner, max_imfs, FIF_REGIME_AUTO);
}

fif_status fif_plan_create_ex(fif_plan_t* out, int64_t n, int64_t batch, fif_dtype dtype, fif_window window,
                              double xi, double delta, int32_t max_inner, int32_t max_imfs, fif_regime regime) {
  if (!out) return FIF_ERR_INVALID_ARG;
  *out = nullptr;
  if (n < 9 || batch < 0 || !(xi > 0.0) || !isfinite(xi) || !(delta > 0.0) || !isfinite(delta) || max_inner < 1 ||
      max_imfs < 1 || (dtype != FIF_F64 && dtype != FIF_F32) ||
      (window != FIF_WINDOW_TRI_SQ && window != FIF_WINDOW_TRI_SQ_WIDE) ||
      (regime != FIF_REGIME_AUTO && regime != FIF_REGIME_RESIDENT && regime != FIF_REGIME_STREAMED))
    return FIF_ERR_INVALID_ARG;
  if (n % 2 != 0) return FIF_ERR_UNSUPPORTED_N;
  const int64_t NC = n / 2;
  const bool resident_ok = (NC & (NC - 1)) == 0 && NC >= 256 && NC <= 4096;
  int reg;
  if (regime == FIF_REGIME_RESIDENT) {
    if (!resident_ok) return FIF_ERR_UNSUPPORTED_N;
    reg = 0;
  } else if (regime == FIF_REGIME_STREAMED) {
    reg = 1;
  } else {
    reg = resident_ok ? 0 : 1;
  }
  if (reg == 1) {  // host-side check of the streamed factorisation before any CUDA call
    st::Geo g;
    if (!st_geometry(n, dtype == FIF_F64, g)) return FIF_ERR_UNSUPPORTED_N;
  }
  fif_plan_s* p = new fif_plan_s();
  p->n = n; p->batch = batch; p->dtype = dtype; p->window = window; p->xi = xi; p->delta = delta;
  p->max_inner = max_inner; p->max_imfs = max_imfs; p->NC = (int)(NC < (1 << 30) ? NC : 0); p->regime = reg;
  if (cudaGetDevice(&p->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device) != cudaSuccess) {
    free_plan(p);
    return FIF_ERR_CUDA;
  }
  if (reg == 1) {
    fif_status st = dtype == FIF_F64 ? st_setup<double>(p) : st_setup<float>(p);
    if (st != FIF_OK) { free_plan(p); return st; }
    *out = p;
    return FIF_OK;
  }
  fif_status st = dtype == FIF_F64 ? upload_tables<double>(p) : upload_tables<float>(p);
  if (st != FIF_OK) { free_plan(p); return st; }
  cudaError_t ce = cudaSuccess;
  dispatch(dtype, p->NC, [&](auto inst) {
    using I = decltype(inst);
    ce = I::prepare();
    p->occ = I::occupancy();
    p->block = I::K::T;
    p->smem = I::K::smem_bytes;
  });
  if (ce != cudaSuccess || p->occ < 1) {
    fprintf(stderr, "fif: kernel setup failed: %s (occ %d)\n", cudaGetErrorString(ce), p->occ);
    free_plan(p);
    return FIF_ERR_CUDA;
  }
  *out = p;
  return FIF_OK;
}

fif_status fif_decompose(fif_plan_t p, const void* d_signals, void* d_imfs, int32_t* d_imf_count,
                         int32_t* d_filter_len, int32_t* d_iters, void* stream) {
  if (!p) return FIF_ERR_INVALID_ARG;
  if (p->batch == 0) return FIF_OK;
  if (!d_signals || !d_imfs || !d_imf_count || !d_filter_len || !d_iters) return FIF_ERR_INVALID_ARG;
  if (((uintptr_t)d_signals | (uintptr_t)d_imfs) & 15) return FIF_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->regime == 1) {
    if (p->dtype == FIF_F64) st_decompose<double>(p, d_signals, d_imfs, d_imf_count, d_filter_len, d_iters, p->batch, s);
    else st_decompose<float>(p, d_signals, d_imfs, d_imf_count, d_filter_len, d_iters, p->batch, s);
    return launch_status();
  }
  dispatch(p->dtype, p->NC, [&](auto inst) {
    using I = decltype(inst);
    I::decompose(p, d_signals, d_imfs, d_imf_count, d_filter_len, d_iters, p->batch, s);
  });
  return launch_status();
}

fif_status fif_decompose_host(fif_plan_t p, const void* h_signals, void* h_imfs, int32_t* h_imf_count,
                              int32_t* h_filter_len, int32_t* h_iters, void* stream) {
  if (!p) return FIF_ERR_INVALID_ARG;
  if (p->batch == 0) return FIF_OK;
  if (!h_signals || !h_imfs || !h_imf_count || !h_filter_len || !h_iters) return FIF_ERR_INVALID_ARG;
  const size_t es = elem_size(p->dtype);
  const size_t in_sig = (size_t)p->n * es, out_sig = in_sig * (size_t)(p->max_imfs + 1);
  const size_t meta_sig = (size_t)(1 + 2 * p->max_imfs);
  if (p->nstages == 0) {
    // chunks of ~1/8 of the batch (>= one full wave of CTAs when possible), 3 stages in flight
    int64_t chunk = (p->batch + 7) / 8;
    const int64_t wave = (int64_t)p->num_sms * p->occ;
    if (chunk < wave) chunk = wave < p->batch ? wave : p->batch;
    p->chunk = chunk;
    p->nstages = (int)((p->batch + chunk - 1) / chunk < FIF_MAX_STAGES ? (p->batch + chunk - 1) / chunk
                                                                        : FIF_MAX_STAGES);
    for (int i = 0; i < p->nstages; ++i) {
      Staging& S = p->st[i];
      if (cudaMalloc(&S.d_in, in_sig * chunk) != cudaSuccess || cudaMalloc(&S.d_out, out_sig * chunk) != cudaSuccess ||
          cudaMalloc(&S.d_meta, sizeof(int32_t) * meta_sig * chunk) != cudaSuccess)
        return FIF_ERR_OOM;
      if (cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&S.done, cudaEventDisableTiming) != cudaSuccess)
        return FIF_ERR_CUDA;
    }
  }
  cudaStream_t user = (cudaStream_t)stream;
  cudaEvent_t start;
  cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  cudaEventRecord(start, user);
  for (int i = 0; i < p->nstages; ++i) cudaStreamWaitEvent(p->st[i].stream, start, 0);
  const int64_t nchunks = (p->batch + p->chunk - 1) / p->chunk;
  for (int64_t c = 0; c < nchunks; ++c) {
    Staging& S = p->st[c % p->nstages];
    const int64_t b0 = c * p->chunk, nb = (b0 + p->chunk <= p->batch) ? p->chunk : p->batch - b0;
    int32_t* d_cnt = S.d_meta;
    int32_t* d_len = S.d_meta + nb;
    int32_t* d_it = d_len + nb * p->max_imfs;
    cudaMemcpyAsync(S.d_in, (const char*)h_signals + b0 * in_sig, nb * in_sig, cudaMemcpyHostToDevice, S.stream);
    if (p->regime == 1) {
      if (p->dtype == FIF_F64) st_decompose<double>(p, S.d_in, S.d_out, d_cnt, d_len, d_it, nb, S.stream);
      else st_decompose<float>(p, S.d_in, S.d_out, d_cnt, d_len, d_it, nb, S.stream);
    } else {
      dispatch(p->dtype, p->NC, [&](auto inst) {
        using I = decltype(inst);
        I::decompose(p, S.d_in, S.d_out, d_cnt, d_len, d_it, nb, S.stream);
      });
    }
    cudaMemcpyAsync((char*)h_imfs + b0 * out_sig, S.d_out, nb * out_sig, cudaMemcpyDeviceToHost, S.stream);
    cudaMemcpyAsync(h_imf_count + b0, d_cnt, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, S.stream);
    cudaMemcpyAsync(h_filter_len + b0 * p->max_imfs, d_len, sizeof(int32_t) * nb * p->max_imfs,
                    cudaMemcpyDeviceToHost, S.stream);
    cudaMemcpyAsync(h_iters + b0 * p->max_imfs, d_it, sizeof(int32_t) * nb * p->max_imfs, cudaMemcpyDeviceToHost,
                    S.stream);
  }
  for (int i = 0; i < p->nstages; ++i) {
    cudaEventRecord(p->st[i].done, p->st[i].stream);
    cudaStreamWaitEvent(user, p->st[i].done, 0);
  }
  cudaEventDestroy(start);
  fif_status st = launch_status();
  if (st != FIF_OK) return st;
  if (cudaStreamSynchronize(user) != cudaSuccess) return FIF_ERR_CUDA;
  return FIF_OK;
}

fif_status fif_destroy(fif_plan_t p) {
  if (!p) return FIF_OK;
  cudaDeviceSynchronize();
  free_plan(p);
  return FIF_OK;
}

int32_t fif_plan_kernels_per_call(fif_plan_t p) {
  if (!p || p->batch == 0) return 0;
  return p->regime == 1 ? st_kernels_per_call(p) : 1;
}

const char* fif_plan_regime(fif_plan_t p) { return p ? (p->regime == 1 ? "streamed" : "resident") : "none"; }

fif_status fif_plan_launch_config(fif_plan_t p, int32_t* grid, int32_t* block, int32_t* smem_bytes) {
  if (!p) return FIF_ERR_INVALID_ARG;
  const int64_t cap = p->regime == 1 ? (int64_t)p->st_grid : (int64_t)p->num_sms * p->occ;
  if (grid) *grid = (int32_t)(p->batch < cap || p->regime == 1 ? (p->regime == 1 ? cap : p->batch) : cap);
  if (block) *block = p->block;
  if (smem_bytes) *smem_bytes = (int32_t)p->smem;
  return FIF_OK;
}

// ---------------------------------------------------------------- test hooks
#define HOOK_SYNC(s)                                       \
  do {                                                     \
    fif_status st_ = launch_status();                      \
    if (st_ != FIF_OK) return st_;                         \
    if (cudaStreamSynchronize(s) != cudaSuccess) return FIF_ERR_CUDA; \
    return FIF_OK;                                         \
  } while (0)

fif_status fif_test_rfft(fif_plan_t p, int64_t batch, const void* d_in, void* d_out, void* stream) {
  if (!p || batch < 0 || (batch && (!d_in || !d_out))) return FIF_ERR_INVALID_ARG;
  if (!batch) return FIF_OK;
  if (p->regime != 0) return FIF_ERR_UNSUPPORTED_N;  // hooks exercise the resident kernels
  cudaStream_t s = (cudaStream_t)stream;
  dispatch(p->dtype, p->NC, [&](auto inst) { decltype(inst)::test_rfft(p, d_in, d_out, batch, s); });
  HOOK_SYNC(s);
}

fif_status fif_test_irfft(fif_plan_t p, int64_t batch, const void* d_in, void* d_out, void* stream) {
  if (!p || batch < 0 || (batch && (!d_in || !d_out))) return FIF_ERR_INVALID_ARG;
  if (!batch) return FIF_OK;
  if (p->regime != 0) return FIF_ERR_UNSUPPORTED_N;  // hooks exercise the resident kernels
  cudaStream_t s = (cudaStream_t)stream;
  dispatch(p->dtype, p->NC, [&](auto inst) { decltype(inst)::test_irfft(p, d_in, d_out, batch, s); });
  HOOK_SYNC(s);
}

fif_status fif_test_extrema(fif_plan_t p, int64_t batch, const void* d_in, int32_t* d_k, void* stream) {
  if (!p || batch < 0 || (batch && (!d_in || !d_k))) return FIF_ERR_INVALID_ARG;
  if (!batch) return FIF_OK;
  if (p->regime != 0) return FIF_ERR_UNSUPPORTED_N;  // hooks exercise the resident kernels
  cudaStream_t s = (cudaStream_t)stream;
  dispatch(p->dtype, p->NC, [&](auto inst) { decltype(inst)::test_extrema(p, d_in, d_k, batch, s); });
  HOOK_SYNC(s);
}

fif_status fif_test_window_spectrum(fif_plan_t p, int32_t L, void* d_out, void* stream) {
  if (!p || L < 1 || !d_out) return FIF_ERR_INVALID_ARG;
  if (p->regime != 0) return FIF_ERR_UNSUPPORTED_N;
  cudaStream_t s = (cudaStream_t)stream;
  dispatch(p->dtype, p->NC, [&](auto inst) { decltype(inst)::test_window(p, L, d_out, s); });
  HOOK_SYNC(s);
}

fif_status fif_test_inner(fif_plan_t p, int64_t batch, int32_t L, const void* d_in, void* d_imf, int32_t* d_N,
                          void* stream) {
  if (!p || batch < 0 || L < 1 || (batch && (!d_in || !d_imf || !d_N))) return FIF_ERR_INVALID_ARG;
  if (!batch) return FIF_OK;
  if (p->regime != 0) return FIF_ERR_UNSUPPORTED_N;  // hooks exercise the resident kernels
  cudaStream_t s = (cudaStream_t)stream;
  dispatch(p->dtype, p->NC, [&](auto inst) { decltype(inst)::test_inner(p, L, d_in, d_imf, d_N, batch, s); });
  HOOK_SYNC(s);
}

}  // extern "C"
