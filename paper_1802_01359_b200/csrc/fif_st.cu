// fif_st.cu -- host side of the streamed regime (fif_streamed.cuh): geometry, tables, L2 waves and
// the per-IMF kernel sequence.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <type_traits>
#include <utility>
#include <vector>

#include "fif_plan.h"

namespace fifhost {
using namespace fifgpu;
namespace {
// ---------------------------------------------------------------- streamed regime (fif_streamed.cuh)
bool smooth235(int64_t x) {
  if (x < 1) return false;
  for (int f : {2, 3, 5})
    while (x % f == 0) x /= f;
  return x == 1;
}
// radix schedule: powers of two in radix-16 passes, the remainder as one radix-4 or -8 pass (two 8s
// instead of 16 x 2), then 3s and 5s
int radices(int64_t N, int* rad, int maxr) {
  int np = 0, a = 0;
  while (N % 2 == 0) { N /= 2; ++a; }
  if (maxr == 8) {  // radix 2 or 4 first, then 8s
    if (a % 3 == 1) { rad[np++] = 2; a -= 1; }
    if (a % 3 == 2) { rad[np++] = 4; a -= 2; }
    while (a >= 3) { rad[np++] = 8; a -= 3; }
    while (N % 3 == 0) { N /= 3; rad[np++] = 3; }
    while (N % 5 == 0) { N /= 5; rad[np++] = 5; }
    return np;
  }
  if (a % 4 == 1 && a >= 5) { rad[np++] = 8; rad[np++] = 4; a -= 5; }
  else if (a % 4 == 1) { rad[np++] = 2; a -= 1; }
  if (a % 4 == 2) { rad[np++] = 4; a -= 2; }
  if (a % 4 == 3) { rad[np++] = 8; a -= 3; }
  while (a >= 4) { rad[np++] = 16; a -= 4; }
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
}  // namespace
// Multi-level geometry: NC = F_0 ... F_{L-1}; the row level holds a mirror pair of rows (2 F_{L-1}
// complex values per smem buffer), the column levels F_i C_i values with C_i >= 128 B of columns.
bool st_geometry(int64_t n, bool f64, st::Geo& g) {
  const int64_t NC = n / 2;
  const int64_t Emax = f64 ? 2048 : 4096;
  int64_t rowmax = Emax / 2, colmax = Emax / (f64 ? 8 : 16);
  // test-only knobs: smaller level lengths force 3- and 4-level geometries at small n
  if (getenv("FIF_ST_ROWMAX")) rowmax = atoll(getenv("FIF_ST_ROWMAX"));
  if (getenv("FIF_ST_COLMAX")) colmax = atoll(getenv("FIF_ST_COLMAX"));
  // L k mod n is evaluated through fp64 (exact below 2^53: L k < n^2/8), so n <= 2^27
  if (n % 2 || NC < 4 || n > (1LL << 27) || !smooth235(NC)) return false;
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
        lv.np = radices(F[i], lv.rad, f64 ? 8 : 16);  // fp64: no radix 16 (register budget, see cta_fft)
        lv.twoff = twoff;
        twoff += lv.F;
        if (i < L - 1) {
          int64_t cmax = Emax / F[i], C = 1;
          for (int64_t c = cmax < S ? cmax : S; c >= 1; --c)
            if (S % c == 0) { C = c; break; }
          lv.C = (int)C;
          lv.swz = lv.F % (f64 ? 8 : 16) == 0;
          lv.pitch = lv.swz ? lv.F : lv.F + 1;
          lv.tiles = lv.A * S / C;
        } else {
          lv.C = 2;
          lv.swz = lv.F % (f64 ? 8 : 16) == 0;
          lv.pitch = lv.F;
          lv.tiles = 0;
        }
        lv.cs = -1;
        if ((lv.C & (lv.C - 1)) == 0)
          for (lv.cs = 0; (1 << lv.cs) < lv.C; ++lv.cs) {}
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
      g.nbch = g.units;  // one probe CTA per row-pair unit
      int bits = 0;
      while ((1LL << bits) < 2 * n + 1) ++bits;
      g.eb = (bits + 1) / 2;
      return true;
    }
  }
  return false;
}
// row tables of a geometry: utab[u] = (row of base u, row of base (P-u) mod P), rbase[row], rmir[row]
// (same digit arithmetic as st::row_of_base / base_of_row)
fif_status st_row_tables(const st::Geo& g, void** d_utab, void** d_rbase, void** d_rmir) {
  auto row_of_base = [&](int64_t base) {
    int64_t r = 0;
    for (int i = 0; i < g.L - 1; ++i) r += ((base / g.Pd[i]) % g.Fd[i]) * g.Sr[i];
    return r;
  };
  auto base_of_row = [&](int64_t row) {
    int64_t b = 0;
    for (int i = 0; i < g.L - 1; ++i) b += ((row / g.Sr[i]) % g.Fd[i]) * g.Pd[i];
    return b;
  };
  std::vector<int2> ut(g.units);
  for (int64_t u = 0; u < g.units; ++u) ut[u] = int2{(int)row_of_base(u), (int)row_of_base((g.P - u) % g.P)};
  std::vector<int> rb(g.P), rm(g.P);
  for (int64_t r = 0; r < g.P; ++r) {
    rb[r] = (int)base_of_row(r);
    rm[r] = (int)row_of_base((g.P - rb[r]) % g.P);
  }
  auto up = [](void** d, const void* h, size_t bytes) {
    if (cudaMalloc(d, bytes) != cudaSuccess) return FIF_ERR_OOM;
    return cudaMemcpy(*d, h, bytes, cudaMemcpyHostToDevice) == cudaSuccess ? FIF_OK : FIF_ERR_CUDA;
  };
  fif_status st;
  if ((st = up(d_utab, ut.data(), sizeof(int2) * ut.size())) != FIF_OK) return st;
  if ((st = up(d_rbase, rb.data(), sizeof(int) * rb.size())) != FIF_OK) return st;
  return up(d_rmir, rm.data(), sizeof(int) * rm.size());
}
namespace {
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
// Tensor maps for the row-major column tiles (cp.async.bulk.tensor): cuTensorMapEncodeTiled through the
// runtime's driver entry point (no link against libcuda).  The pass's source as a 3-D tensor of 8-byte
// elements {lower index s (S values), digit row a F + f (NC / S rows), slot}: a tile is the box {C, F, 1}.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return (EncodeTiledFn)f;
  }();
  return fn;
}
// box limits of the tensor-map tile of a level (each box side <= 256 elements) and the 128-byte alignment of
// every ring buffer (the shared-memory destination of a tensor copy)
static bool tile_box_ok(const st::Level& lv, size_t vbytes) {
  return lv.C * (vbytes / 8) <= 256 && lv.F <= 256 && (lv.C * vbytes) % 16 == 0 &&
         ((size_t)lv.C * lv.pitch * vbytes) % 128 == 0;
}
static bool tile_map(CUtensorMap* tm, const void* base, const st::Level& lv, size_t vbytes, int64_t NC, int64_t slots,
                     int64_t slot_bytes) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc || !tile_box_ok(lv, vbytes) || ((uintptr_t)base % 16) != 0) return false;
  const cuuint64_t epv = vbytes / 8;
  const cuuint64_t dims[3] = {(cuuint64_t)lv.S * epv, (cuuint64_t)(NC / lv.S), (cuuint64_t)slots};
  const cuuint64_t strides[2] = {(cuuint64_t)lv.S * vbytes, (cuuint64_t)slot_bytes};
  const cuuint32_t box[3] = {(cuuint32_t)(lv.C * epv), (cuuint32_t)lv.F, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// the k_col instance for a column level: its compile-time transform path (st::col_fft CS), 0 = generic
static int col_schedule(const st::Level& lv, bool f64) {
  auto is = [&](int F, std::initializer_list<int> r) {
    if (lv.F != F || !lv.swz || lv.pitch != F || lv.np != (int)r.size()) return false;
    int i = 0;
    for (int x : r)
      if (lv.rad[i++] != x) return false;
    return true;
  };
  if (!f64) {
    if (is(32, {8, 4})) return 1;
    if (is(64, {4, 16})) return 2;
    if (is(128, {8, 16})) return 3;
    if (is(256, {16, 16})) return 4;
    if (lv.F == 12 && !lv.swz && lv.pitch == 13 && lv.np == 2 && lv.rad[0] == 4 && lv.rad[1] == 3) return 9;
    if (lv.F == 20 && !lv.swz && lv.pitch == 21 && lv.np == 2 && lv.rad[0] == 4 && lv.rad[1] == 5) return 10;
  } else {
    if (is(128, {2, 8, 8})) return 5;
    if (is(256, {4, 8, 8})) return 6;
    if (is(32, {4, 8})) return 7;
    if (is(64, {8, 8})) return 8;
  }
  return 0;
}
// the row kernels' instance: 1 = the compile-time full-length row (st::row_fft RS)
static int row_schedule(const st::Level& lv, bool f64) {
  const int F = f64 ? 1024 : 2048;
  const int r64[4] = {2, 8, 8, 8}, r32[3] = {8, 16, 16};
  const int* r = f64 ? r64 : r32;
  const int np = f64 ? 4 : 3;
  if (lv.F != F || !lv.swz || lv.pitch != F || lv.np != np) return 0;
  for (int i = 0; i < np; ++i)
    if (lv.rad[i] != r[i]) return 0;
  return 1;
}
// any level processed as C x F tiles (the distributed passes): column shapes, then the row lengths
int pass_schedule_impl(const st::Level& lv, bool f64) {
  const int cs = col_schedule(lv, f64);
  if (cs) return cs;
  return row_schedule(lv, f64) ? (f64 ? 11 : 12) : 0;
}
template <typename Real, int DIR, int KIND, typename F>
static void for_col_instances(F&& f) {
  f(st::k_col<Real, DIR, KIND, 0>);
  if constexpr (sizeof(Real) == 4) {
    f(st::k_col<Real, DIR, KIND, 1>);
    f(st::k_col<Real, DIR, KIND, 2>);
    f(st::k_col<Real, DIR, KIND, 3>);
    f(st::k_col<Real, DIR, KIND, 4>);
    f(st::k_col<Real, DIR, KIND, 9>);
    f(st::k_col<Real, DIR, KIND, 10>);
    f(st::k_col<Real, DIR, KIND, 21>);
    f(st::k_col<Real, DIR, KIND, 22>);
    f(st::k_col<Real, DIR, KIND, 23>);
    f(st::k_col<Real, DIR, KIND, 24>);
    f(st::k_col<Real, DIR, KIND, 29>);
    f(st::k_col<Real, DIR, KIND, 30>);
  } else {
    f(st::k_col<Real, DIR, KIND, 5>);
    f(st::k_col<Real, DIR, KIND, 6>);
    f(st::k_col<Real, DIR, KIND, 7>);
    f(st::k_col<Real, DIR, KIND, 8>);
    f(st::k_col<Real, DIR, KIND, 25>);
    f(st::k_col<Real, DIR, KIND, 26>);
    f(st::k_col<Real, DIR, KIND, 27>);
    f(st::k_col<Real, DIR, KIND, 28>);
  }
}
template <typename Real, int DIR, int KIND, typename... A>
static void launch_col(int cs, int grid, size_t smem, cudaStream_t s, A... a) {
  switch (cs) {
    case 1: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 1><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 2: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 2><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 3: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 3><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 4: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 4><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 9: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 9><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 10: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 10><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 5: if constexpr (sizeof(Real) == 8) { st::k_col<Real, DIR, KIND, 5><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 6: if constexpr (sizeof(Real) == 8) { st::k_col<Real, DIR, KIND, 6><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 7: if constexpr (sizeof(Real) == 8) { st::k_col<Real, DIR, KIND, 7><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 8: if constexpr (sizeof(Real) == 8) { st::k_col<Real, DIR, KIND, 8><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 21: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 21><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 22: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 22><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 23: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 23><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 24: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 24><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 29: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 29><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 30: if constexpr (sizeof(Real) == 4) { st::k_col<Real, DIR, KIND, 30><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 25: if constexpr (sizeof(Real) == 8) { st::k_col<Real, DIR, KIND, 25><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 26: if constexpr (sizeof(Real) == 8) { st::k_col<Real, DIR, KIND, 26><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 27: if constexpr (sizeof(Real) == 8) { st::k_col<Real, DIR, KIND, 27><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    case 28: if constexpr (sizeof(Real) == 8) { st::k_col<Real, DIR, KIND, 28><<<grid, st::kColThreads, smem, s>>>(a...); return; } break;
    default: break;
  }
  st::k_col<Real, DIR, KIND, 0><<<grid, st::kColThreads, smem, s>>>(a...);
}

template <typename Real>
fif_status st_setup_t(fif_plan_s* p) {
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
  if ((s = st_row_tables(g, &p->d_utab, &p->d_rbase, &p->d_rmir)) != FIF_OK) return s;
  g.utab = (const int2*)p->d_utab;
  g.rbase = (const int*)p->d_rbase;
  g.rmir = (const int*)p->d_rmir;
  // L2 waves: the working set of a signal (spectrum, remainder, IMF slot: 3 n b bytes) of a wave
  // of signals stays in the 126 MB L2 across the passes of an IMF
  const double wave_mb = getenv("FIF_WAVE_MB") ? atof(getenv("FIF_WAVE_MB")) : 1024.0;
  const int64_t per_sig = 3 * p->n * (int64_t)sizeof(Real);
  int64_t wave = (int64_t)(wave_mb * 1048576.0 / (double)per_sig);
  if (wave < 1) wave = 1;
  const int64_t B = p->batch > 0 ? p->batch : 1;
  if (wave > B) wave = B;
  p->st_wave = wave;
  const size_t ni = (size_t)B * 13 + 2 * (size_t)B;  // + slist, scnt, pmax (B doubles)
  const size_t segb = (size_t)B * g.nseg * (sizeof(uint32_t) + 2 * sizeof(Real));
  const size_t grpb = (size_t)B * g.ngrp * (sizeof(uint32_t) + 2 * sizeof(Real));
  const size_t redb = (size_t)B * g.nbch * 2 * st::kProbes * sizeof(double);
  // workspace layout: two spectrum buffers (X_in / X_out ping-pong per IMF: the speculative damping
  // keeps X_in intact), their Nyquist bins, the control block, and (spectral-peak rule) the power array
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  p->ws_ctl_bytes = ni * sizeof(int32_t) + segb + grpb + redb + 256;
  p->ws_xn = up(2 * sizeof(V) * B * g.NC);
  p->ws_ctl = p->ws_xn + up(2 * sizeof(V) * B);
  p->ws_pnat = p->ws_ctl + up(p->ws_ctl_bytes);
  p->ws_end = p->ws_pnat;
  p->ws_end_pnat = p->ws_pnat + up(sizeof(double) * B * (size_t)(g.NC + 1));
  if ((s = st_bind_workspace(p, nullptr, 0)) != FIF_OK) return s;
  // shared memory and grids
  for (int i = 0; i < g.L - 1; ++i)  // three tile buffers + the level's twiddles
    p->st_smem_col[i] = 3 * sizeof(V) * (size_t)g.lv[i].C * g.lv[i].pitch + sizeof(V) * (size_t)g.lv[i].F;
  p->st_smem_rows = 2 * sizeof(V) * 2 * (size_t)g.lv[g.L - 1].pitch;
  p->st_smem_rows_inv = 3 * sizeof(V) * 2 * (size_t)g.lv[g.L - 1].pitch;  // two staging buffers + the FFT's
  size_t smax = p->st_smem_rows_inv;
  for (int i = 0; i < g.L - 1; ++i) smax = smax > p->st_smem_col[i] ? smax : p->st_smem_col[i];
  cudaError_t e = cudaSuccess;
  auto attr = [&](auto kern) {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
  };
  for_col_instances<Real, -1, st::PASS_FWD_FIRST>(attr);
  for_col_instances<Real, -1, st::PASS_MID>(attr);
  for_col_instances<Real, 1, st::PASS_MID>(attr);
  for_col_instances<Real, 1, st::PASS_INV_LAST>(attr);
  for (int i = 0; i < g.L - 1; ++i) p->st_col_cs[i] = col_schedule(g.lv[i], sizeof(Real) == 8);
  // Row-major column tiles staged by the TMA engine, for a compile-time schedule and 16-byte aligned rows (row
  // length, digit stride and signal length multiples of 16 bytes).  Same arithmetic in the same order as the
  // cp.async tiles (bit-identical decompositions, tests/test_gpu_streamed.py).  FIF_ST_RM=1: one cp.async.bulk per
  // tile row (measured slower than cp.async: many short row copies per tile).
  // FIF_ST_RM=2: the same tiles landed by ONE cp.async.bulk.tensor each (a 3-D box of a tensor map encoded per
  // call over the pass's source), when the level's box fits the tensor-map limits.
  // Default (FIF_ST_RM unset): the tensor-map tiles (measured faster on every geometry of configs 2-4, DESIGN.md
  // §8); FIF_ST_RM=0 forces the cp.async tiles, 1 the row-by-row bulk copies.
  const char* rmenv = getenv("FIF_ST_RM");
  const int rm_mode = rmenv ? atoi(rmenv) : 2;
  const bool rm_on = rm_mode == 1 || rm_mode == 2;
  const bool tm_on = rm_mode == 2 && encode_tiled() != nullptr;
  for (int i = 0; i < g.L - 1; ++i) {
    const st::Level& lv = g.lv[i];
    const bool ok = p->st_col_cs[i] >= 1 && p->st_col_cs[i] <= 10 && (lv.C * sizeof(V)) % 16 == 0 &&
                    (lv.S * sizeof(V)) % 16 == 0 && (g.n * sizeof(Real)) % 16 == 0;
    p->st_col_rm[i] = rm_on && ok ? p->st_col_cs[i] + 20 : 0;
    p->st_col_tm[i] = p->st_col_rm[i] && tm_on && tile_box_ok(lv, sizeof(V)) ? 1 : 0;
  }
  attr(st::k_rows_fwd<Real, 0>);
  attr(st::k_rows_fwd<Real, 1>);
  attr(st::k_rows_inv<Real, 0, 0, 0>);
  attr(st::k_rows_inv<Real, kFastCap, 0, 0>);
  attr(st::k_rows_inv<Real, 0, 1, 0>);
  attr(st::k_rows_inv<Real, kFastCap, 1, 0>);
  attr(st::k_rows_inv<Real, 0, 0, 1>);
  attr(st::k_rows_inv<Real, kFastCap, 0, 1>);
  attr(st::k_rows_inv<Real, 0, 1, 1>);
  attr(st::k_rows_inv<Real, kFastCap, 1, 1>);
  p->st_row_rs = row_schedule(g.lv[g.L - 1], sizeof(Real) == 8);
  if (e != cudaSuccess) {
    fprintf(stderr, "fif: streamed setup failed: %s\n", cudaGetErrorString(e));
    return FIF_ERR_CUDA;
  }
  {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, st::k_col<Real, 1, st::PASS_INV_LAST>, st::kColThreads, smax);
    p->st_grid_col = p->num_sms * (occ > 0 ? occ : 1);
  }
  p->st_grid_rows = p->st_row_rs ? occ_grid(p, st::k_rows_inv<Real, kFastCap, 1, 1>, p->st_smem_rows_inv)
                                 : occ_grid(p, st::k_rows_inv<Real, kFastCap, 1, 0>, p->st_smem_rows_inv);
  p->st_grid_probe = occ_grid(p, st::k_probe<Real, kFastCap, 1>, 0);
  p->st_grid = p->st_grid_rows;
  for (int i = 0; i < 2; ++i)
    if (cudaStreamCreateWithFlags(&p->st_streams[i], cudaStreamNonBlocking) != cudaSuccess) return FIF_ERR_CUDA;
  for (int i = 0; i < 3; ++i)
    if (cudaEventCreateWithFlags(&p->st_ev[i], cudaEventDisableTiming) != cudaSuccess) return FIF_ERR_CUDA;
  p->block = st::kThreads;
  p->smem = smax;
  p->occ = 1;
  return FIF_OK;
}

// Ctl / geometry of the wave of signals [b0, b0 + nb)
st::Ctl ctl_at(const st::Ctl& c, const st::Geo& g, int64_t b0, size_t rsz) {
  st::Ctl r = c;
  r.k += b0; r.L += b0; r.N += b0; r.M += b0; r.active += b0; r.search += b0; r.lo += b0; r.hi += b0;
  r.bad += b0; r.cnt += b0; r.redo += b0; r.pmax += b0; r.slist += b0; r.scnt += b0;
  r.segi += b0 * g.nseg;
  r.segv = (char*)c.segv + b0 * g.nseg * 2 * rsz;
  r.gi += b0 * g.ngrp;
  r.gv = (char*)c.gv + b0 * g.ngrp * 2 * rsz;
  r.red += b0 * g.nbch * 2 * st::kProbes;
  return r;
}
int grid_for(int64_t work, int cap) { return (int)(work < cap ? (work > 0 ? work : 1) : cap); }
int capped(const fif_plan_s* p, int g) { return p->grid_cap > 0 && p->grid_cap < g ? p->grid_cap : g; }

// the whole decomposition as stream-ordered kernels (no host synchronisation), one L2 wave at a time
template <typename Real>
void st_decompose_t(fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its, int64_t batch,
                    int64_t boff, cudaStream_t s) {
  using V = typename Cx<Real>::V;
  const int TB = st::kThreads;
  const st::Tabs<Real> tb{(const double2*)p->d_Eh, (const double2*)p->d_El, (const V*)p->d_Th, (const V*)p->d_Tl,
                          (const V*)p->d_twl};
  // waves alternate between two internal streams (independent signals: their latency-bound kernels
  // overlap), joined back into the caller's stream at the end
  const int64_t nw = (batch + p->st_wave - 1) / p->st_wave;
  const int nstream = nw > 1 ? 2 : 1;
  cudaStream_t user = s;
  if (nstream > 1) {
    cudaEventRecord(p->st_ev[0], user);
    for (int i = 0; i < 2; ++i) cudaStreamWaitEvent(p->st_streams[i], p->st_ev[0], 0);
  }
  for (int64_t b0 = 0, w = 0; b0 < batch; b0 += p->st_wave, ++w) {
    s = nstream > 1 ? p->st_streams[w & 1] : user;
    st::Geo g = p->geo;
    g.batch = batch - b0 < p->st_wave ? batch - b0 : p->st_wave;
    g.stop = p->stop;
    g.delta = p->delta;
    g.gamma = p->gamma;
    g.mask = p->mask;
    g.pnat = p->d_pnat ? (double*)p->d_pnat + (boff + b0) * (g.NC + 1) : nullptr;
    const st::Ctl c = ctl_at(p->ctl, g, boff + b0, sizeof(Real));
    const Real* sg = (const Real*)sig + b0 * g.n;
    Real* out = (Real*)imfs + b0 * g.sig_stride;
    const int64_t Bp = p->batch > 0 ? p->batch : 1;
    V* X = (V*)p->d_X + (boff + b0) * g.NC;        // X_0 (forward transform output)
    V* Xn = (V*)p->d_Xn + boff + b0;
    V* Xalt = (V*)p->d_X + (Bp + boff + b0) * g.NC;  // X_1
    V* Xnalt = (V*)p->d_Xn + Bp + boff + b0;
    int32_t* ln = lens + b0 * g.max_imfs;
    int32_t* it = its + b0 * g.max_imfs;
    const int Lv = g.L;
    const bool fast = g.max_inner == kFastCap;
    const st::Level& top = g.lv[Lv - 1];
    const int gcol = capped(p, p->st_grid_col), grow = grid_for(g.batch * g.units, capped(p, p->st_grid_rows));
    const int gprobe = grid_for(g.batch * g.nbch, capped(p, p->st_grid_probe));
    const int gfold = grid_for(g.batch * g.ngrp, capped(p, p->num_sms * 4));
    const int gsig = (int)((g.batch + TB - 1) / TB);
    auto col = [&](int i) { return grid_for(g.batch * g.lv[i].tiles, gcol); };
    // the column passes' instance: row-major bulk-copy tiles when the level and this call's buffers allow
    const bool aligned16 = ((uintptr_t)sg % 16) == 0 && ((uintptr_t)out % 16) == 0;
    auto ccs = [&](int i) { return aligned16 && p->st_col_rm[i] ? p->st_col_rm[i] : p->st_col_cs[i]; };
    // tensor maps of this wave's sources (tile = one box): the signals (level 0 forward), X (the other forward
    // levels), the IMF slots of d_imfs (inverse levels); a level whose map cannot be encoded copies row by row
    CUtensorMap tmf[st::kMaxLev] = {}, tmi[st::kMaxLev] = {};
    int tmf_on[st::kMaxLev] = {}, tmi_on[st::kMaxLev] = {};
    for (int i = 0; i < Lv - 1; ++i) {
      if (!(aligned16 && p->st_col_rm[i] && p->st_col_tm[i])) continue;
      tmf_on[i] = i == 0 ? tile_map(&tmf[i], sg, g.lv[i], sizeof(V), g.NC, g.batch, g.n * (int64_t)sizeof(Real))
                         : tile_map(&tmf[i], X, g.lv[i], sizeof(V), g.NC, g.batch, g.NC * (int64_t)sizeof(V));
      tmi_on[i] = tile_map(&tmi[i], out, g.lv[i], sizeof(V), g.NC, g.batch * (g.max_imfs + 1),
                           g.n * (int64_t)sizeof(Real));
    }
    Nvtx wave("streamed/wave");
    st::k_init<<<gsig, TB, 0, s>>>(g, c);
    launch_col<Real, -1, st::PASS_FWD_FIRST>(ccs(0), col(0), p->st_smem_col[0], s, g, g.lv[0], g.lv[0], sg, out, X, tb, c, tmf[0], tmf_on[0]);
    st::k_fold<Real><<<gfold, TB, 0, s>>>(g, c, 0, ln, it);
    for (int i = 1; i < Lv - 1; ++i)
      launch_col<Real, -1, st::PASS_MID>(ccs(i), col(i), p->st_smem_col[i], s, g, g.lv[i], g.lv[i], sg, out, X, tb, c, tmf[i], tmf_on[i]);
    if (p->st_row_rs) st::k_rows_fwd<Real, 1><<<grow, TB, p->st_smem_rows, s>>>(g, top, X, Xn, tb, c);
    else st::k_rows_fwd<Real, 0><<<grow, TB, p->st_smem_rows, s>>>(g, top, X, Xn, tb, c);
    auto peaks = [&](const V* Xs, const V* Xns) {  // spectral-peak rule: L for the next IMF
      if (!g.mask) return;
      st::k_peak1<Real><<<grow, TB, 0, s>>>(g, Xs, Xns, c);
      st::k_peak2<Real><<<grow, TB, 0, s>>>(g, c);
    };
    peaks(X, Xn);
    for (int m = 0; m < g.max_imfs; ++m) {
      Nvtx imf("streamed/imf");
      V* Xi = (m & 1) ? Xalt : X;
      V* Xo = (m & 1) ? X : Xalt;
      V* Xni = (m & 1) ? Xnalt : Xn;
      V* Xno = (m & 1) ? Xn : Xnalt;
      // the K-ary rounds and the redo touch only the few signals whose SD(cap) <= delta: one CTA per
      // (signal, unit) so that the others cost a flag load and an exit, not a serial skip loop
      const int gall = (int)(g.batch * g.units < (1LL << 30) ? g.batch * g.units : (1LL << 30));
      (void)gall;
      auto rows = [&](auto spec, auto cap, int redo_only) {
        if (p->st_row_rs)
          st::k_rows_inv<Real, decltype(cap)::value, decltype(spec)::value, 1>
              <<<grow, TB, p->st_smem_rows_inv, s>>>(g, top, g.lv[Lv - 2], out, Xi, Xo, Xni, Xno, tb, c, redo_only);
        else
          st::k_rows_inv<Real, decltype(cap)::value, decltype(spec)::value, 0>
              <<<grow, TB, p->st_smem_rows_inv, s>>>(g, top, g.lv[Lv - 2], out, Xi, Xo, Xni, Xno, tb, c, redo_only);
      };
      auto probe = [&](auto cap, auto mode) {
        st::k_probe<Real, decltype(cap)::value, decltype(mode)::value><<<gprobe, TB, 0, s>>>(g, Xi, Xni, tb, c);
      };
      using F0 = std::integral_constant<int, 0>;
      using F1 = std::integral_constant<int, 1>;
      using FC = std::integral_constant<int, kFastCap>;
      if (g.stop == 0) {
        // SD rule: fused cap probe + speculative damping; K-ary search and a redo only if SD(cap) <= delta
        if (fast) rows(F1{}, FC{}, 0); else rows(F1{}, F0{}, 0);
        for (int r = 0; r < p->st_rounds; ++r) probe(F0{}, F1{});
        if (fast) rows(F0{}, FC{}, 1); else rows(F0{}, F0{}, 1);
      } else {
        // a-priori N0 rule: one max-reduction probe decides N, then the damping
        if (fast) probe(FC{}, F0{}); else probe(F0{}, F0{});
        if (fast) rows(F0{}, FC{}, 0); else rows(F0{}, F0{}, 0);
      }
      for (int i = Lv - 2; i >= 1; --i)
        launch_col<Real, 1, st::PASS_MID>(ccs(i), col(i), p->st_smem_col[i], s, g, g.lv[i], g.lv[i - 1], sg, out, X, tb, c, tmi[i], tmi_on[i]);
      launch_col<Real, 1, st::PASS_INV_LAST>(ccs(0), col(0), p->st_smem_col[0], s, g, g.lv[0], g.lv[0], sg, out, X, tb, c, tmi[0], tmi_on[0]);
      st::k_fold<Real><<<gfold, TB, 0, s>>>(g, c, 1, ln, it);
      peaks(Xo, Xno);
    }
    st::k_final<Real><<<grid_for(g.batch, p->num_sms * 4), TB, 0, s>>>(g, out, c, cnt + b0, ln, it);
  }
  if (nstream > 1)
    for (int i = 0; i < 2; ++i) {
      cudaEventRecord(p->st_ev[1 + i], p->st_streams[i]);
      cudaStreamWaitEvent(user, p->st_ev[1 + i], 0);
    }
}
}  // namespace
int pass_schedule(const st::Level& lv, bool f64) { return pass_schedule_impl(lv, f64); }
int st_kernels_per_call(const fif_plan_s* p) {
  const int L = p->geo.L;
  const int64_t waves = p->batch > 0 ? (p->batch + p->st_wave - 1) / p->st_wave : 0;
  const int per_imf = (p->stop == 0 ? (p->st_rounds + L + 2) : (L + 2)) + (p->mask ? 2 : 0);
  return (int)(waves * (2 + (L - 1) + 1 + (p->mask ? 2 : 0) + p->max_imfs * per_imf + 1));
}

size_t st_workspace_bytes(const fif_plan_s* p) { return p->mask ? p->ws_end_pnat : p->ws_end; }

// Carve d_X, d_Xn, the control block (zeroed: the state a fresh plan starts from) and, with the
// spectral-peak rule, d_pnat out of one block: the caller's (base != nullptr, >= bytes needed) or a
// plan-owned allocation.  No decompose on the plan may be pending.
fif_status st_bind_workspace(fif_plan_s* p, void* base, size_t bytes) {
  const size_t need = st_workspace_bytes(p);
  if (base && bytes < need) return FIF_ERR_INVALID_ARG;
  if (cudaDeviceSynchronize() != cudaSuccess) return FIF_ERR_CUDA;
  // the new block first: on failure the plan keeps its current (valid) workspace and buffers
  void* own = nullptr;
  if (!base) {
    if (cudaMalloc(&own, need) != cudaSuccess) {
      cudaGetLastError();
      return FIF_ERR_OOM;
    }
    base = own;
  }
  cudaFree(p->d_ws_own);
  p->d_ws_own = own;
  p->d_ws_user = own ? nullptr : base;
  p->ws_user_bytes = own ? 0 : bytes;
  char* w = (char*)base;
  p->d_X = w;
  p->d_Xn = w + p->ws_xn;
  p->d_ctl = w + p->ws_ctl;
  p->d_pnat = p->mask ? (void*)(w + p->ws_pnat) : nullptr;
  const st::Geo& g = p->geo;
  const int64_t B = p->batch > 0 ? p->batch : 1;
  const size_t rs = p->dtype == FIF_F64 ? sizeof(double) : sizeof(float);
  const size_t ni = (size_t)B * 13 + 2 * (size_t)B;
  char* q = (char*)p->d_ctl;
  auto take = [&](size_t nb) {
    char* r = q;
    q += (nb + 15) & ~(size_t)15;
    return (void*)r;
  };
  st::Ctl& c = p->ctl;
  c.red = (double*)take((size_t)B * g.nbch * 2 * st::kProbes * sizeof(double));
  c.segv = take((size_t)B * g.nseg * 2 * rs);
  c.gv = take((size_t)B * g.ngrp * 2 * rs);
  c.segi = (uint32_t*)take((size_t)B * g.nseg * sizeof(uint32_t));
  c.gi = (uint32_t*)take((size_t)B * g.ngrp * sizeof(uint32_t));
  int32_t* ip = (int32_t*)take(ni * sizeof(int32_t));
  c.k = ip; c.L = ip + B; c.N = ip + 2 * B; c.M = ip + 3 * B; c.active = ip + 4 * B; c.search = ip + 5 * B;
  c.lo = ip + 6 * B; c.hi = ip + 7 * B; c.bad = ip + 8 * B; c.cnt = (uint32_t*)(ip + 9 * B); c.redo = ip + 10 * B;
  c.slist = ip + 11 * B; c.scnt = ip + 12 * B;
  c.pmax = (double*)take((size_t)B * sizeof(double));
  if (cudaMemset(p->d_ctl, 0, p->ws_ctl_bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    return FIF_ERR_CUDA;
  return FIF_OK;
}

fif_status st_setup(fif_plan_s* p) { return p->dtype == FIF_F64 ? st_setup_t<double>(p) : st_setup_t<float>(p); }
void st_decompose(fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its,
                  int64_t batch, int64_t boff, cudaStream_t s) {
  if (p->dtype == FIF_F64) st_decompose_t<double>(p, sig, imfs, cnt, lens, its, batch, boff, s);
  else st_decompose_t<float>(p, sig, imfs, cnt, lens, its, batch, boff, s);
}
void st_free(fif_plan_s* p) {
  cudaFree(p->d_Eh);
  cudaFree(p->d_El);
  cudaFree(p->d_Th);
  cudaFree(p->d_Tl);
  cudaFree(p->d_twl);
  cudaFree(p->d_ws_own);  // (a caller workspace stays the caller's)
  cudaFree(p->d_utab);
  cudaFree(p->d_rbase);
  cudaFree(p->d_rmir);
  for (int i = 0; i < 2; ++i)
    if (p->st_streams[i]) cudaStreamDestroy(p->st_streams[i]);
  for (int i = 0; i < 3; ++i)
    if (p->st_ev[i]) cudaEventDestroy(p->st_ev[i]);
}
}  // namespace fifhost
