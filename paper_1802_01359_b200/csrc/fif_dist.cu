// fif_dist.cu -- the distributed regime: ONE long signal (BASELINE config 3, n = 2^26) time-block
// sharded over P GPUs (rank r owns samples [r n/P, (r+1) n/P)), one process per GPU, NCCL over
// NVLink for the exchange steps.
//
// Transform (z_m = x_2m + i x_2m+1, NC = n/2 = P Q complex points, rank r holding z[r Q, (r+1) Q)):
// the outermost FFT digit is the rank.  Forward: all-to-all #1 (rank r sends slice q of its block to
// rank q), length-P DFTs over the rank digit + twiddle e^{-2 pi i s k0/NC}, all-to-all #2 (block k0
// to rank k0), then a local Q-point multi-level FFT (the streamed regime's passes).  Rank r then
// holds the bins k = r + P j ("cyclic"), j in digit-reversed local order.  The Hermitian partner
// NC - k of its bins lives on rank (P - r) mod P: one partner exchange after the forward transform
// gives every rank an aligned copy Xm of its partners' spectrum, which it then damps locally every
// IMF with the same a^N -- so the per-IMF real-IFFT pre-processing (X_k with X_{NC-k}) needs no
// communication.
// Per IMF:  probe sums (local) -> allgather -> every rank folds them in rank
// order and takes the same decision (N);  damping + pre-processing (local);  local inverse passes;
// twiddle, all-to-all #3, length-P IDFTs, all-to-all #4 back to the time-block layout;  IMF store,
// R -= IMF, local extrema partial -> allgather -> ordered fold (boundary differences between
// ranks included) -> k, L (identical on every rank).
//
// Collectives go through a small interface with two implementations: NCCL (libnccl.so.2 loaded at
// run time) and an emulation that runs all P ranks of one process on the current device back to
// back, the collectives becoming device copies (tests and single-GPU runs of the same algorithm).
#include <dlfcn.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include <nccl.h>
#include "fif_plan.h"

using namespace fifgpu;

namespace fifgpu {
namespace ds {
using st::Level;
using st::Mono;
using st::kThreads;
using st::kNW;
using st::kProbes;

constexpr int kMaxP = 64;

struct DGeo {
  st::Geo g;         // global n, NC, eb, window/xi/delta; lv[], Frow, P (= local rows), Fd/Pd/Sr: local Q-point FFT
  int64_t Q;         // local complex points = NC / P
  int P, rank;
  int64_t segc;      // complex points per extrema segment
  int64_t nseg;      // local segments
  int64_t nloc;      // local reals = 2 Q
};

struct DExt {      // a rank's extrema partial (ordered monoid of its block) + bad-sample flag
  double first, last;
  uint32_t mono;
  int32_t bad;
  int64_t pad;
};

struct DCtl {
  int32_t* s;        // [16] scalars: k, L, N, M, active, search, lo, hi, bad, cnt
  uint32_t* segi;    // [nseg]
  double* segv;      // [nseg][2]
  DExt* ext_send;    // [1]
  DExt* ext_recv;    // [P]
  double* red;       // [nblk][2 kProbes] per-CTA probe partials
  double* pr_send;   // [2 kProbes]
  double* pr_recv;   // [P][2 kProbes]
};
enum { S_K = 0, S_L, S_N, S_M, S_ACT, S_SEARCH, S_LO, S_HI, S_BAD, S_CNT };

template <typename Real>
using Tabs = st::Tabs<Real>;

// position of local bin j's partner for rank 0 (partner j' = (Q - j) mod Q) -- the single-GPU
// mirror structure of the local Q-point FFT
__device__ __forceinline__ int64_t partner_pos0(const st::Geo& g, int64_t pos) {
  const int F = g.Frow;
  const int64_t row = pos / F;
  const int t = (int)(pos - row * F);
  if (__ldg(g.rbase + row) == 0) return (t == 0 ? 0 : F - t);
  return (int64_t)__ldg(g.rmir + row) * F + (F - 1 - t);
}
__device__ __forceinline__ int64_t local_bin(const st::Geo& g, int64_t pos) {
  const int F = g.Frow;
  const int64_t row = pos / F;
  return __ldg(g.rbase + row) + g.P * (pos - row * F);
}

// ---------------------------------------------------------------- local multi-level passes (in place)
// Level tile = C consecutive lower indices x F digit values; DIR -1 forward (DFT, twiddle),
// +1 inverse (conjugate twiddle, IDFT).  Twiddles use the global-n table (E2 = 2n/(F S)).
template <typename Real, int DIR, int CS = 0>
__global__ void __launch_bounds__(kThreads, FIF_ST_MINB) k_d_pass(const __grid_constant__ DGeo d,
                                                        const __grid_constant__ Level lv,
                                                        typename Cx<Real>::V* __restrict__ buf,
                                                        const __grid_constant__ Tabs<Real> tb,
                                                        const int32_t* __restrict__ s) {
  using V = typename Cx<Real>::V;
  if (!s[S_ACT] && DIR > 0) return;
  extern __shared__ __align__(16) char smem_raw[];
  V* A = reinterpret_cast<V*>(smem_raw);
  V* Bf = A + (size_t)lv.C * lv.pitch;
  const int64_t spt = lv.S / lv.C;
  for (int64_t t = blockIdx.x; t < lv.tiles; t += gridDim.x) {
    const int64_t a = t / spt, s0 = (t - a * spt) * lv.C;
    const int64_t base = a * (int64_t)lv.F * lv.S + s0;
    const int FC = lv.F * lv.C;
    constexpr int U = st::TileCap<Real>::value / kThreads;
    V v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {  // unconditional (clamped) loads keep v[] in registers
      const int i = threadIdx.x + j * kThreads;
      int f, cc;
      st::tile_fc(lv, i < FC ? i : 0, f, cc);
      v[j] = buf[base + (int64_t)f * lv.S + cc];
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = threadIdx.x + j * kThreads;
      if (i < FC) {
        int f, cc;
        st::tile_fc(lv, i, f, cc);
        V x = v[j];
        if (DIR > 0 && lv.S > 1) x = cmul(x, st::Er(tb, d.g.eb, lv.E2 * (s0 + cc) * f));
        A[st::sidx<V>(cc, f, lv.pitch, lv.swz)] = x;
      }
    }
    Level lvs = lv;  // the transform path of this instance (pass_schedule); twiddles pre-offset
    lvs.twoff = 0;
    V* out = st::col_fft<DIR, V, CS>(A, Bf, lvs, lv.C, tb.tw + lv.twoff);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = threadIdx.x + j * kThreads;
      if (i < FC) {
        int f, cc;
        st::tile_fc(lv, i, f, cc);
        V x = out[st::sidx<V>(cc, f, lv.pitch, lv.swz)];
        if (DIR < 0 && lv.S > 1) x = cmul(x, cconj(st::Er(tb, d.g.eb, lv.E2 * (s0 + cc) * f)));
        buf[base + (int64_t)f * lv.S + cc] = x;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- cross-rank digit: length-P DFTs
// in [m0][s'] (P x Q/P) -> out [k0][s'] = sum_m0 in[m0][s'] e^{DIR 2 pi i m0 k0/P}, forward with the
// twiddle e^{-2 pi i s k0/NC} (s = rank Q/P + s') applied after.
// With `peer` (a table of the P ranks' receive buffers), output chunk k0 is stored straight into rank
// k0's buffer at [rank Q/P + s'] over NVLink -- the all-to-all that follows the DFT fused into it.
template <typename Real, int DIR>
__global__ void __launch_bounds__(kThreads) k_d_rankdft(const __grid_constant__ DGeo d,
                                                        const typename Cx<Real>::V* __restrict__ in,
                                                        typename Cx<Real>::V* __restrict__ out,
                                                        const __grid_constant__ Tabs<Real> tb,
                                                        const int32_t* __restrict__ s,
                                                        typename Cx<Real>::V* const* __restrict__ peer = nullptr) {
  using V = typename Cx<Real>::V;
  if (DIR > 0 && !s[S_ACT]) return;
  const int64_t W = d.Q / d.P;
  const int P = d.P;
  const int64_t stepP = 2 * d.g.n / P;  // E index of e^{i 2 pi / P}
  for (int64_t sp = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sp < W; sp += (int64_t)gridDim.x * blockDim.x) {
    V x[kMaxP];
    for (int m = 0; m < P; ++m) x[m] = in[(int64_t)m * W + sp];
    const int64_t sglob = (int64_t)d.rank * W + sp;
    for (int k0 = 0; k0 < P; ++k0) {
      V acc = x[0];
      for (int m = 1; m < P; ++m) {
        V w = st::Er(tb, d.g.eb, stepP * ((m * k0) % P));
        if (DIR < 0) w = cconj(w);
        acc = cadd(acc, cmul(x[m], w));
      }
      if (DIR < 0) acc = cmul(acc, cconj(st::Er(tb, d.g.eb, 4 * sglob * k0)));  // 2n/NC = 4
      if (peer) peer[k0][(int64_t)d.rank * W + sp] = acc;
      else out[(int64_t)k0 * W + sp] = acc;
    }
  }
  if (peer) __threadfence_system();
}

// signal slices straight into the ranks' receive buffers (the forward all-to-all #1 as peer stores)
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_d_scatter(const __grid_constant__ DGeo d,
                                                        const typename Cx<Real>::V* __restrict__ z,
                                                        typename Cx<Real>::V* const* __restrict__ peer) {
  const int64_t W = d.Q / d.P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.Q; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = i / W;
    peer[q][(int64_t)d.rank * W + (i - q * W)] = z[i];
  }
  __threadfence_system();
}

// inverse level-0 twiddle: out[s] = in[s] e^{+2 pi i s rank/NC}
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_d_twiddle_inv(const __grid_constant__ DGeo d,
                                                            const typename Cx<Real>::V* __restrict__ in,
                                                            typename Cx<Real>::V* __restrict__ out,
                                                            const __grid_constant__ Tabs<Real> tb,
                                                            const int32_t* __restrict__ s) {
  if (!s[S_ACT]) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.Q; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = cmul(in[i], st::Er(tb, d.g.eb, 4 * i * d.rank));
}
// ... fused with the all-to-all #3: slice q of the twiddled block into rank q's buffer at [rank Q/P + s']
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_d_twiddle_scatter(const __grid_constant__ DGeo d,
                                                                const typename Cx<Real>::V* __restrict__ in,
                                                                typename Cx<Real>::V* const* __restrict__ peer,
                                                                const __grid_constant__ Tabs<Real> tb,
                                                                const int32_t* __restrict__ s) {
  if (!s[S_ACT]) return;
  const int64_t W = d.Q / d.P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.Q; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = i / W;
    peer[q][(int64_t)d.rank * W + (i - q * W)] = cmul(in[i], st::Er(tb, d.g.eb, 4 * i * d.rank));
  }
  __threadfence_system();
}

// ---------------------------------------------------------------- extrema partials (contiguous segments)
// src: Q complex (natural local order); segment = segc complex points = 2 segc reals
template <typename Real>
__device__ void seg_partials(const DGeo& d, const typename Cx<Real>::V* src, DCtl c) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwg = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nd = 2 * d.segc - 1;
  const int64_t q = (nd + 31) / 32;
  for (int64_t sg = gw; sg < d.nseg; sg += nwg) {
    const typename Cx<Real>::V* v = src + sg * d.segc;
    Mono m{0, 0, 0};
    const int64_t d0 = lane * q, d1 = min(d0 + q, nd);
    if (d0 < d1) {
      auto x_at = [&](int64_t j) -> Real { const auto z = v[j >> 1]; return (j & 1) ? z.y : z.x; };
      Real prev = x_at(d0);
      for (int64_t j = d0; j < d1; ++j) {
        const Real x = x_at(j + 1);
        m = st::mcomb(m, st::mdiff<Real>(x - prev));
        prev = x;
      }
    }
    m = st::warp_mono(m);
    if (lane == 0) {
      c.segi[sg] = st::mpack(m);
      c.segv[2 * sg] = (double)v[0].x;
      c.segv[2 * sg + 1] = (double)v[d.segc - 1].y;
    }
  }
}

// a1 input: R = s (local trend slot), non-finite flag, extrema partials of s
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_d_load(const __grid_constant__ DGeo d, const Real* __restrict__ sig,
                                                     Real* __restrict__ R, DCtl c) {
  using V = typename Cx<Real>::V;
  const V* z = reinterpret_cast<const V*>(sig);
  V* Rv = reinterpret_cast<V*>(R);
  bool finite = true;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.Q; i += (int64_t)gridDim.x * blockDim.x) {
    const V v = z[i];
    finite &= isfinite((double)v.x) && isfinite((double)v.y);
    Rv[i] = v;
  }
  if (!finite) atomicOr(c.s + S_BAD, 1);
  seg_partials<Real>(d, z, c);
}

// a6 epilogue: IMF slot M <- z (natural local order), R -= IMF, extrema partials of the new R
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_d_epi(const __grid_constant__ DGeo d,
                                                    const typename Cx<Real>::V* __restrict__ z, Real* __restrict__ imfs,
                                                    DCtl c) {
  using V = typename Cx<Real>::V;
  if (!c.s[S_ACT]) return;
  V* imf = reinterpret_cast<V*>(imfs + (int64_t)c.s[S_M] * d.nloc);
  V* R = reinterpret_cast<V*>(imfs + (int64_t)d.g.max_imfs * d.nloc);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.Q; i += (int64_t)gridDim.x * blockDim.x) {
    const V v = z[i];
    __stcs(imf + i, v);
    R[i] = csub(R[i], v);
  }
}
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_d_segs(const __grid_constant__ DGeo d, const Real* __restrict__ imfs,
                                                     DCtl c) {
  if (!c.s[S_ACT]) return;
  seg_partials<Real>(d, reinterpret_cast<const typename Cx<Real>::V*>(imfs + (int64_t)d.g.max_imfs * d.nloc), c);
}

// local ordered fold of the segment partials -> this rank's DExt (one CTA)
__global__ void __launch_bounds__(kThreads) k_d_fold_local(const __grid_constant__ DGeo d, DCtl c, int first) {
  __shared__ Mono sm[kNW];
  if (!first && !c.s[S_ACT]) return;
  const Mono m = st::fold_items<double>(c.segi, c.segv, 0, d.nseg, sm);
  if (threadIdx.x == 0) {
    DExt e;
    e.first = c.segv[0];
    e.last = c.segv[2 * (d.nseg - 1) + 1];
    e.mono = st::mpack(m);
    e.bad = c.s[S_BAD];
    e.pad = 0;
    *c.ext_send = e;
  }
}

// fold the P rank partials in rank order (boundary differences between blocks included), then
// decide.  mode 0: after loading s (k of s, non-finite check); mode 1: after IMF M (bookkeeping).
__global__ void k_d_decide_ext(const __grid_constant__ DGeo d, DCtl c, int mode, int32_t* __restrict__ lens,
                               int32_t* __restrict__ iters) {
  if (threadIdx.x || blockIdx.x) return;
  int32_t* s = c.s;
  if (mode == 1 && !s[S_ACT]) return;
  Mono acc{0, 0, 0};
  int bad = 0;
  double prev = 0.0;
  for (int r = 0; r < d.P; ++r) {
    const DExt e = c.ext_recv[r];
    if (r > 0) acc = st::mcomb(acc, st::mdiff<double>(e.first - prev));
    acc = st::mcomb(acc, st::munpack(e.mono));
    prev = e.last;
    bad |= e.bad;
  }
  int M = s[S_M];
  if (mode == 0) {
    if (bad) {
      s[S_M] = -1;
      s[S_ACT] = 0;
      return;
    }
  } else {
    lens[M] = 2 * s[S_L];
    iters[M] = s[S_N];
    s[S_M] = ++M;
  }
  s[S_K] = acc.c;
  if (acc.c < 2 || M >= d.g.max_imfs) {
    s[S_ACT] = 0;
  } else {
    s[S_L] = st::filter_half_length(d.g, acc.c);
    s[S_SEARCH] = 0;
  }
}

// ---------------------------------------------------------------- forward post-processing
// X[pos] = X_k = E + e^{-2 pi i k/n} O, Xm[pos] = X_{NC-k} = conj(E - e^{-2 pi i k/n} O) from Z = Y[pos]
// and its partner Z_{NC-k} (rank 0: local; rank P/2: local reversed; others: the partner rank's
// array, received in Zp, reversed).  k = 0: X_0 = Re Z_0 + Im Z_0, Xm = X_NC = Re Z_0 - Im Z_0.
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_d_post(const __grid_constant__ DGeo d,
                                                     const typename Cx<Real>::V* __restrict__ Y,
                                                     const typename Cx<Real>::V* __restrict__ Zp,
                                                     typename Cx<Real>::V* __restrict__ X,
                                                     typename Cx<Real>::V* __restrict__ Xm,
                                                     const __grid_constant__ Tabs<Real> tb, const int32_t* s) {
  using V = typename Cx<Real>::V;
  if (!s[S_ACT]) return;
  const int r = d.rank, P = d.P;
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < d.Q;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const V Pv = Y[pos];
    V Qv;
    if (r == 0) Qv = Y[partner_pos0(d.g, pos)];
    else if (2 * r == P) Qv = Y[d.Q - 1 - pos];
    else Qv = Zp[d.Q - 1 - pos];
    const int64_t k = r + (int64_t)P * local_bin(d.g, pos);
    if (k == 0) {
      X[pos] = V{Pv.x + Pv.y, (Real)0};
      Xm[pos] = V{Pv.x - Pv.y, (Real)0};
      continue;
    }
    const Real h = (Real)0.5;
    const V E = V{h * (Pv.x + Qv.x), h * (Pv.y - Qv.y)};
    const V D = V{h * (Pv.x - Qv.x), h * (Pv.y + Qv.y)};
    const V O = V{D.y, -D.x};
    const V TO = cmul(cconj(st::Er(tb, d.g.eb, 2 * k)), O);
    X[pos] = cadd(E, TO);
    Xm[pos] = cconj(csub(E, TO));
  }
}

// ---------------------------------------------------------------- a5 probes (local sums + rank fold)
template <typename Real, int CAP, int MODE>
__global__ void __launch_bounds__(kThreads, MODE == 1 ? FIF_PROBE1_MINB : 3) k_d_probe(const __grid_constant__ DGeo d,
                                                         const typename Cx<Real>::V* __restrict__ X,
                                                         const typename Cx<Real>::V* __restrict__ Xm,
                                                         const __grid_constant__ Tabs<Real> tb, DCtl c) {
  using V = typename Cx<Real>::V;
  constexpr int NV = MODE == 0 ? 2 : 2 * kProbes;
  __shared__ double sred[kNW][NV];
  __shared__ int last;
  const int32_t* s = c.s;
  if (!s[S_ACT] || (MODE == 1 && !s[S_SEARCH])) return;
  const int L = s[S_L];
  int N0, step;
  if (MODE == 0) {
    N0 = d.g.max_inner; step = 0;
  } else {
    const int lo = s[S_LO], hi = s[S_HI];
    step = (hi - lo + kProbes) / (kProbes + 1);
    if (step < 1) step = 1;
    N0 = lo + step;
  }
  const double invn = 1.0 / (double)d.g.n;
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = 0.0;
  const bool useMax = MODE == 0 && d.g.stop == 1;
  auto add = [&](const V& x, double w, double cw) {
    const double pk = cw * ((double)x.x * (double)x.x + (double)x.y * (double)x.y);
    const double a = 1.0 - w;
    if (useMax) {  // N0 rule: max |X_k|^2
      acc[0] = fmax(acc[0], pk / cw);
    } else if constexpr (MODE == 0) {
      double e = (CAP > 0 && N0 == CAP) ? st::upow_c<(CAP > 0 ? CAP - 1 : 1)>(a) : st::upow_rt(a, N0 - 1);
      e *= e;
      acc[0] += pk * e;
      acc[1] += pk * w * w * e;
    } else {
      const double a2 = a * a;
      double y = st::upow_rt(a2, N0 - 1);
      const double z = st::upow_rt(a2, step);
      const double qk = pk * w * w;
#pragma unroll
      for (int q = 0; q < kProbes; ++q) {
        acc[2 * q] += pk * y;
        acc[2 * q + 1] += qk * y;
        y *= z;
      }
    }
  };
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < d.Q;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = d.rank + (int64_t)d.P * local_bin(d.g, pos);
    double wk, wm;
    st::what_pair(d.g, tb, L, invn, k, wk, wm);
    add(X[pos], wk, k == 0 ? 1.0 : 2.0);
    if (k == 0) add(Xm[pos], wm, 1.0);  // the Nyquist bin X_NC lives in Xm on rank 0
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double v = acc[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, v, o);
      v = useMax ? fmax(v, u) : v + u;
    }
    if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5][i] = v;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double v = 0.0;
    for (int w = 0; w < kNW; ++w) v = useMax ? fmax(v, sred[w][threadIdx.x]) : v + sred[w][threadIdx.x];
    c.red[(int64_t)blockIdx.x * (2 * kProbes) + threadIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(reinterpret_cast<unsigned*>(c.s + S_CNT), 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x < NV) {  // this rank's partial: CTA partials in block order
    __threadfence();
    double v = 0.0;
    for (unsigned bq = 0; bq < gridDim.x; ++bq) {
      const double u = __ldcg(c.red + (int64_t)bq * (2 * kProbes) + threadIdx.x);
      v = useMax ? fmax(v, u) : v + u;
    }
    c.pr_send[threadIdx.x] = v;
    if (threadIdx.x == 0) c.s[S_CNT] = 0;
  }
}

// every rank sums the P partials in rank order and takes the same decision
template <int MODE>
__global__ void k_d_decide_probe(const __grid_constant__ DGeo d, DCtl c) {
  if (threadIdx.x || blockIdx.x) return;
  int32_t* s = c.s;
  if (!s[S_ACT] || (MODE == 1 && !s[S_SEARCH])) return;
  constexpr int NV = MODE == 0 ? 2 : 2 * kProbes;
  double PQ[NV];
  const bool useMax = MODE == 0 && d.g.stop == 1;
  for (int i = 0; i < NV; ++i) {
    double v = 0.0;
    for (int r = 0; r < d.P; ++r) v = useMax ? fmax(v, c.pr_recv[r * (2 * kProbes) + i]) : v + c.pr_recv[r * (2 * kProbes) + i];
    PQ[i] = v;
  }
  if (useMax) {  // N = min(N0, cap) from the global max |X_k|^2 (A16-A18)
    const double rhs = d.g.delta / (sqrt(PQ[0] / (double)d.g.n) * sqrt((double)(d.g.n - 1)));
    s[S_N] = n0_capped(rhs, d.g.max_inner);
    s[S_SEARCH] = 0;
  } else if (MODE == 0) {
    s[S_N] = d.g.max_inner;
    if (PQ[1] <= d.g.delta2 * PQ[0]) {
      s[S_LO] = 0;
      s[S_HI] = d.g.max_inner;
      s[S_SEARCH] = d.g.max_inner > 1 ? 1 : 0;
      if (d.g.max_inner == 1) s[S_N] = 1;
    }
  } else {
    const int lo = s[S_LO], hi = s[S_HI];
    int step = (hi - lo + kProbes) / (kProbes + 1);
    if (step < 1) step = 1;
    int nlo = lo, nhi = hi;
    for (int q = 0; q < kProbes; ++q) {
      const int Nq = lo + step * (q + 1);
      if (Nq >= hi) break;
      if (PQ[2 * q + 1] <= d.g.delta2 * PQ[2 * q]) { nhi = Nq; break; }
      nlo = Nq;
    }
    s[S_LO] = nlo;
    s[S_HI] = nhi;
    if (nhi - nlo <= 1) {
      s[S_SEARCH] = 0;
      s[S_N] = nhi;
    }
  }
}

// ---------------------------------------------------------------- a6 damping + pre-processing (local)
template <typename Real, int CAP>
__global__ void __launch_bounds__(kThreads, 3) k_d_pre(const __grid_constant__ DGeo d,
                                                       typename Cx<Real>::V* __restrict__ X,
                                                       typename Cx<Real>::V* __restrict__ Xm,
                                                       typename Cx<Real>::V* __restrict__ W,
                                                       const __grid_constant__ Tabs<Real> tb, const int32_t* s) {
  using V = typename Cx<Real>::V;
  if (!s[S_ACT]) return;
  const int L = s[S_L], N = s[S_N];
  const double invn = 1.0 / (double)d.g.n;
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < d.Q;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = d.rank + (int64_t)d.P * local_bin(d.g, pos);
    double wk, wm;
    st::what_pair(d.g, tb, L, invn, k, wk, wm);
    double dk, dm;
    if (CAP > 0 && N == CAP) {
      dk = st::upow_c<(CAP > 0 ? CAP : 1)>(1.0 - wk);
      dm = st::upow_c<(CAP > 0 ? CAP : 1)>(1.0 - wm);
    } else {
      dk = st::upow_rt(1.0 - wk, N);
      dm = st::upow_rt(1.0 - wm, N);
    }
    if (d.g.gamma > 0.0) {  // gamma-threshold (A19)
      if (dk >= 1.0 - d.g.gamma) dk = 1.0;
      if (dm >= 1.0 - d.g.gamma) dm = 1.0;
    }
    const V xk = X[pos], xm = Xm[pos];
    const V Av = cscale(xk, (Real)(dk * invn)), Bv = cscale(xm, (Real)(dm * invn));
    const V S = V{Av.x + Bv.x, Av.y - Bv.y};
    const V D = V{Av.x - Bv.x, Av.y + Bv.y};
    const V T = mul_i<1>(cmul(st::Er(tb, d.g.eb, 2 * k), D));
    W[pos] = cadd(S, T);
    X[pos] = cscale(xk, (Real)(1.0 - dk));
    Xm[pos] = cscale(xm, (Real)(1.0 - dm));
  }
}

// ---------------------------------------------------------------- a7 final (local slots; replicated ints)
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_d_final(const __grid_constant__ DGeo d, Real* __restrict__ imfs,
                                                      const int32_t* s, int32_t* count, int32_t* lens,
                                                      int32_t* iters) {
  const int M = s[S_M];
  const int64_t nl = d.nloc, tot = (int64_t)(d.g.max_imfs + 1) * nl;
  const Real* R = imfs + (int64_t)d.g.max_imfs * nl;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st_ = (int64_t)gridDim.x * blockDim.x;
  if (M < 0) {
    for (int64_t i = i0; i < tot; i += st_) imfs[i] = (Real)0;
  } else if (M < d.g.max_imfs) {
    Real* tr = imfs + (int64_t)M * nl;
    for (int64_t i = i0; i < nl; i += st_) tr[i] = R[i];
  }
  if (blockIdx.x == 0) {
    for (int m = threadIdx.x; m < d.g.max_imfs; m += blockDim.x)
      if (m >= M) { lens[m] = 0; iters[m] = 0; }
    if (threadIdx.x == 0) *count = M;
  }
}
// zero the slots past the trend (after k_d_final has copied R into slot M)
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_d_zero(const __grid_constant__ DGeo d, Real* __restrict__ imfs,
                                                     const int32_t* s) {
  const int M = s[S_M];
  if (M < 0 || M >= d.g.max_imfs) return;
  const int64_t nl = d.nloc;
  for (int64_t i = (int64_t)(M + 1) * nl + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       i < (int64_t)(d.g.max_imfs + 1) * nl; i += (int64_t)gridDim.x * blockDim.x)
    imfs[i] = (Real)0;
}

__global__ void k_d_init(int32_t* s) {
  if (threadIdx.x < 16) s[threadIdx.x] = 0;
  if (threadIdx.x == 0) s[S_ACT] = 1;
}

}  // namespace ds
}  // namespace fifgpu

// ================================================================== host side
namespace fifhost {
namespace {
using namespace fifgpu::ds;

// NCCL loaded at run time (the library does not link it: resident / streamed plans never need it)
struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  decltype(&ncclCommGetAsyncError) commGetAsyncError = nullptr;
  bool load() {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      fprintf(stderr, "fif: dlopen(libnccl.so.2) failed: %s\n", dlerror());
      return false;
    }
#define FIF_SYM(f, n) f = (decltype(f))dlsym(h, n)
    FIF_SYM(getUniqueId, "ncclGetUniqueId");
    FIF_SYM(commInitRank, "ncclCommInitRank");
    FIF_SYM(commDestroy, "ncclCommDestroy");
    FIF_SYM(allGather, "ncclAllGather");
    FIF_SYM(allReduce, "ncclAllReduce");
    FIF_SYM(send, "ncclSend");
    FIF_SYM(recv, "ncclRecv");
    FIF_SYM(groupStart, "ncclGroupStart");
    FIF_SYM(groupEnd, "ncclGroupEnd");
    FIF_SYM(errStr, "ncclGetErrorString");
    FIF_SYM(commGetAsyncError, "ncclCommGetAsyncError");
#undef FIF_SYM
    return getUniqueId && commInitRank && commDestroy && allGather && allReduce && send && recv && groupStart &&
           groupEnd && commGetAsyncError;
  }
};
Nccl& nccl() {
  static Nccl n;
  return n;
}

// one rank's device state
struct DRank {
  DGeo d;
  void *X = nullptr, *Xm = nullptr, *T = nullptr, *U = nullptr;  // Q complex each
  void* small = nullptr;
  DCtl c{};
};

template <typename T>
size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

struct DistPlan {
  int P = 1, rank = 0;           // this process's rank (NCCL) ; emulated: all ranks local
  bool emulated = false;
  ncclComm_t comm = nullptr;
  std::vector<DRank> ranks;      // 1 (NCCL) or P (emulated)
  void *Eh = nullptr, *El = nullptr, *Th = nullptr, *Tl = nullptr, *tw = nullptr;
  void *utab = nullptr, *rbase = nullptr, *rmir = nullptr;
  size_t smem_pass[st::kMaxLev] = {};
  int pass_cs[st::kMaxLev] = {};  // compile-time transform path per level (k_d_pass CS)
  int grid_pass = 0, grid_elem = 0, grid_probe = 0;
  int rounds = 0;
  int64_t Q = 0;
  // peer mode (FIF_DIST_PEER=1): the all-to-alls fused into the producing kernels as NVLink peer
  // stores into the ranks' buffers (CUDA IPC handles in a multi-process plan), a barrier after each
  bool peer = false;
  void* dpeer = nullptr;                 // device: [local ranks][2][P] pointers (U table, T table)
  std::vector<void*> hpeer;              // host copy of the same table (read by the host launch code)
  std::vector<void*> ipc_open;           // IPC-mapped peer buffers to close
  void* dbar = nullptr;                  // one int for the NCCL barrier
};

namespace {

fif_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return FIF_OK;
  fprintf(stderr, "fif: %s failed: %s\n", what, nccl().errStr ? nccl().errStr(r) : "?");
  return FIF_ERR_NCCL;
}

// ncclCommGetAsyncError polling (network / peer failures are reported asynchronously by NCCL)
fif_status async_error(DistPlan& D) {
  if (D.emulated || !D.comm || !nccl().commGetAsyncError) return FIF_OK;
  ncclResult_t ae = ncclSuccess;
  ncclResult_t r = nccl().commGetAsyncError(D.comm, &ae);
  if (r != ncclSuccess) return nccl_check(r, "ncclCommGetAsyncError");
  if (ae != ncclSuccess && ae != ncclInProgress) return nccl_check(ae, "NCCL communicator (async error)");
  return FIF_OK;
}

// ---------------- collectives (NCCL or emulated copies); `field` selects the per-rank buffer
template <typename F1, typename F2>
fif_status c_allgather(DistPlan& D, F1 send, F2 recv, size_t bytes, cudaStream_t s) {
  if (D.emulated) {
    for (int dst = 0; dst < D.P; ++dst)
      for (int src = 0; src < D.P; ++src)
        cudaMemcpyAsync((char*)recv(dst, D.ranks[dst]) + src * bytes, send(src, D.ranks[src]), bytes,
                        cudaMemcpyDeviceToDevice, s);
    return FIF_OK;
  }
  return nccl_check(nccl().allGather(send(0, D.ranks[0]), recv(0, D.ranks[0]), bytes, ncclUint8, D.comm, s),
                    "ncclAllGather");
}
// all-to-all: chunk q (bytes each) of rank r's send buffer -> chunk r of rank q's receive buffer
template <typename F1, typename F2>
fif_status c_alltoall(DistPlan& D, F1 send, F2 recv, size_t bytes, cudaStream_t s) {
  if (D.emulated) {
    for (int dst = 0; dst < D.P; ++dst)
      for (int src = 0; src < D.P; ++src)
        cudaMemcpyAsync((char*)recv(dst, D.ranks[dst]) + src * bytes,
                        (const char*)send(src, D.ranks[src]) + dst * bytes, bytes, cudaMemcpyDeviceToDevice, s);
    return FIF_OK;
  }
  fif_status st = nccl_check(nccl().groupStart(), "ncclGroupStart");
  for (int q = 0; q < D.P && st == FIF_OK; ++q) {
    st = nccl_check(nccl().send((const char*)send(0, D.ranks[0]) + q * bytes, bytes, ncclUint8, q, D.comm, s),
                    "ncclSend");
    if (st == FIF_OK)
      st = nccl_check(nccl().recv((char*)recv(0, D.ranks[0]) + q * bytes, bytes, ncclUint8, q, D.comm, s), "ncclRecv");
  }
  fif_status st2 = nccl_check(nccl().groupEnd(), "ncclGroupEnd");
  return st != FIF_OK ? st : st2;
}
// partner exchange: rank r's send buffer -> rank (P - r) mod P's receive buffer (self-partners skip)
template <typename F1, typename F2>
fif_status c_partner(DistPlan& D, F1 send, F2 recv, size_t bytes, cudaStream_t s) {
  if (D.emulated) {
    for (int r = 0; r < D.P; ++r) {
      const int p = (D.P - r) % D.P;
      if (p != r) cudaMemcpyAsync(recv(p, D.ranks[p]), send(r, D.ranks[r]), bytes, cudaMemcpyDeviceToDevice, s);
    }
    return FIF_OK;
  }
  const int p = (D.P - D.rank) % D.P;
  if (p == D.rank) return FIF_OK;
  fif_status st = nccl_check(nccl().groupStart(), "ncclGroupStart");
  if (st == FIF_OK) st = nccl_check(nccl().send(send(0, D.ranks[0]), bytes, ncclUint8, p, D.comm, s), "ncclSend");
  if (st == FIF_OK) st = nccl_check(nccl().recv(recv(0, D.ranks[0]), bytes, ncclUint8, p, D.comm, s), "ncclRecv");
  fif_status st2 = nccl_check(nccl().groupEnd(), "ncclGroupEnd");
  return st != FIF_OK ? st : st2;
}

int gmin(int64_t work, int cap) { return (int)(work < cap ? (work > 0 ? work : 1) : cap); }

// k_d_pass instance for a level's transform path (pass_schedule in fif_st.cu)
template <typename Real, int DIR, typename F>
static void for_dpass_instances(F&& f) {
  f(k_d_pass<Real, DIR, 0>);
  if constexpr (sizeof(Real) == 4) {
    f(k_d_pass<Real, DIR, 1>); f(k_d_pass<Real, DIR, 2>); f(k_d_pass<Real, DIR, 3>); f(k_d_pass<Real, DIR, 4>);
    f(k_d_pass<Real, DIR, 9>); f(k_d_pass<Real, DIR, 10>); f(k_d_pass<Real, DIR, 12>);
  } else {
    f(k_d_pass<Real, DIR, 5>); f(k_d_pass<Real, DIR, 6>); f(k_d_pass<Real, DIR, 7>); f(k_d_pass<Real, DIR, 8>);
    f(k_d_pass<Real, DIR, 11>);
  }
}
template <typename Real, int DIR, typename... A>
static void launch_dpass(int cs, int64_t grid, size_t smem, cudaStream_t s, A... a) {
#define FIF_DP(C, COND)                                                        \
  case C:                                                                      \
    if constexpr (COND) {                                                      \
      k_d_pass<Real, DIR, C><<<(unsigned)grid, kThreads, smem, s>>>(a...);     \
      return;                                                                  \
    }                                                                          \
    break;
  constexpr bool f32 = sizeof(Real) == 4, f64 = sizeof(Real) == 8;
  switch (cs) {
    FIF_DP(1, f32) FIF_DP(2, f32) FIF_DP(3, f32) FIF_DP(4, f32) FIF_DP(9, f32) FIF_DP(10, f32) FIF_DP(12, f32)
    FIF_DP(5, f64) FIF_DP(6, f64) FIF_DP(7, f64) FIF_DP(8, f64) FIF_DP(11, f64)
    default: break;
  }
#undef FIF_DP
  k_d_pass<Real, DIR, 0><<<(unsigned)grid, kThreads, smem, s>>>(a...);
}

template <typename Real>
fif_status dist_setup_t(fif_plan_s* p, DistPlan& D) {
  using V = typename Cx<Real>::V;
  const int64_t n = p->n, NC = n / 2;
  const int P = D.P;
  const int64_t Q = NC / P;
  D.Q = Q;
  // local Q-point FFT geometry (levels of the streamed regime; the row level is a plain C = 1 level here)
  st::Geo lg;
  if (!st_geometry(2 * Q, sizeof(Real) == 8, lg)) return FIF_ERR_UNSUPPORTED_N;
  st::Geo g = lg;
  g.n = n;
  g.NC = NC;
  g.batch = 1;
  g.max_imfs = p->max_imfs; g.max_inner = p->max_inner; g.window = (int)p->window;
  g.xi = p->xi; g.delta2 = p->delta * p->delta;
  g.sig_stride = 0;
  int bits = 0;
  while ((1LL << bits) < 2 * n + 1) ++bits;
  g.eb = (bits + 1) / 2;
  for (int i = 0; i < g.L; ++i) {
    st::Level& lv = g.lv[i];
    lv.E2 = 2 * n / ((int64_t)lv.F * lv.S);
    if (i == g.L - 1) {
      lv.C = 1;
      lv.cs = 0;
      lv.pitch = lv.swz ? lv.F : lv.F + 1;
      lv.tiles = lv.A;
    }
  }
  // tables: e^{i pi j/n} for the global n, per-level Stockham twiddles
  const long double PI = 3.141592653589793238462643383279502884L;
  const int64_t nh = (2 * n >> g.eb) + 1, nl = 1LL << g.eb;
  std::vector<double2> Eh(nh), El(nl);
  std::vector<V> Th(nh), Tl(nl), tw;
  for (int64_t h = 0; h < nh; ++h) {
    const long double a = PI * (long double)(h << g.eb) / (long double)n;
    Eh[h] = double2{(double)cosl(a), (double)sinl(a)};
    Th[h] = V{(Real)cosl(a), (Real)sinl(a)};
  }
  for (int64_t l = 0; l < nl; ++l) {
    const long double a = PI * (long double)l / (long double)n;
    El[l] = double2{(double)cosl(a), (double)sinl(a)};
    Tl[l] = V{(Real)cosl(a), (Real)sinl(a)};
  }
  for (int i = 0; i < g.L; ++i)
    for (int j = 0; j < g.lv[i].F; ++j) {
      const long double th = 2.0L * PI * (long double)j / (long double)g.lv[i].F;
      tw.push_back(V{(Real)cosl(th), (Real)(-sinl(th))});
    }
  auto up = [](void** dp, const void* hp, size_t bytes) {
    if (cudaMalloc(dp, bytes) != cudaSuccess) return FIF_ERR_OOM;
    return cudaMemcpy(*dp, hp, bytes, cudaMemcpyHostToDevice) == cudaSuccess ? FIF_OK : FIF_ERR_CUDA;
  };
  fif_status s;
  if ((s = up(&D.Eh, Eh.data(), sizeof(double2) * nh)) != FIF_OK) return s;
  if ((s = up(&D.El, El.data(), sizeof(double2) * nl)) != FIF_OK) return s;
  if ((s = up(&D.Th, Th.data(), sizeof(V) * nh)) != FIF_OK) return s;
  if ((s = up(&D.Tl, Tl.data(), sizeof(V) * nl)) != FIF_OK) return s;
  if ((s = up(&D.tw, tw.data(), sizeof(V) * tw.size())) != FIF_OK) return s;
  if ((s = st_row_tables(g, &D.utab, &D.rbase, &D.rmir)) != FIF_OK) return s;
  g.utab = (const int2*)D.utab;
  g.rbase = (const int*)D.rbase;
  g.rmir = (const int*)D.rmir;
  // launch shapes
  size_t smax = 0;
  for (int i = 0; i < g.L; ++i) {
    D.smem_pass[i] = 2 * sizeof(V) * (size_t)g.lv[i].C * g.lv[i].pitch;
    smax = smax > D.smem_pass[i] ? smax : D.smem_pass[i];
  }
  cudaError_t e = cudaSuccess;
  auto attr = [&](auto kern) {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
  };
  for_dpass_instances<Real, -1>(attr);
  for_dpass_instances<Real, 1>(attr);
  if (e != cudaSuccess) return FIF_ERR_CUDA;
  for (int i = 0; i < g.L; ++i) D.pass_cs[i] = pass_schedule(g.lv[i], sizeof(Real) == 8);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_d_pass<Real, 1>, kThreads, smax);
  D.grid_pass = p->num_sms * (occ > 0 ? occ : 1);
  D.grid_elem = p->num_sms * 8;
  D.grid_probe = p->num_sms * 3;
  if (p->grid_cap > 0) {  // test knob (FIF_GRID_CAP): other CTA schedules, same bits
    D.grid_pass = D.grid_pass < p->grid_cap ? D.grid_pass : p->grid_cap;
    D.grid_elem = D.grid_elem < p->grid_cap ? D.grid_elem : p->grid_cap;
    D.grid_probe = D.grid_probe < p->grid_cap ? D.grid_probe : p->grid_cap;
  }
  D.rounds = 0;
  for (int64_t len = p->max_inner; len > 1; len = (len + kProbes) / (kProbes + 1)) ++D.rounds;
  // per-rank buffers
  const int nloc = D.emulated ? P : 1;
  D.ranks.resize(nloc);
  for (int li = 0; li < nloc; ++li) {
    DRank& R = D.ranks[li];
    R.d.g = g;
    R.d.Q = Q;
    R.d.P = P;
    R.d.rank = D.emulated ? li : D.rank;
    R.d.nloc = 2 * Q;
    R.d.segc = Q < 2048 ? Q : 2048;
    while (Q % R.d.segc) --R.d.segc;
    R.d.nseg = Q / R.d.segc;
    const size_t qb = sizeof(V) * (size_t)Q;
    if (cudaMalloc(&R.X, qb) != cudaSuccess || cudaMalloc(&R.Xm, qb) != cudaSuccess ||
        cudaMalloc(&R.T, qb) != cudaSuccess || cudaMalloc(&R.U, qb) != cudaSuccess)
      return FIF_ERR_OOM;
    const size_t b_s = al<int>(16 * 4), b_segi = al<int>(R.d.nseg * 4), b_segv = al<int>(R.d.nseg * 16),
                 b_ext = al<int>(sizeof(DExt)), b_extr = al<int>(sizeof(DExt) * P),
                 b_red = al<int>((size_t)D.grid_probe * 2 * kProbes * 8), b_pr = al<int>(2 * kProbes * 8),
                 b_prr = al<int>((size_t)P * 2 * kProbes * 8);
    const size_t tot = b_s + b_segi + b_segv + b_ext + b_extr + b_red + b_pr + b_prr;
    if (cudaMalloc(&R.small, tot) != cudaSuccess) return FIF_ERR_OOM;
    if (cudaMemset(R.small, 0, tot) != cudaSuccess) return FIF_ERR_CUDA;
    char* q = (char*)R.small;
    R.c.s = (int32_t*)q; q += b_s;
    R.c.segi = (uint32_t*)q; q += b_segi;
    R.c.segv = (double*)q; q += b_segv;
    R.c.ext_send = (DExt*)q; q += b_ext;
    R.c.ext_recv = (DExt*)q; q += b_extr;
    R.c.red = (double*)q; q += b_red;
    R.c.pr_send = (double*)q; q += b_pr;
    R.c.pr_recv = (double*)q; q += b_prr;
  }
  p->block = kThreads;
  p->smem = smax;
  p->occ = occ;
  return FIF_OK;
}

// Peer mode: per local rank a device table [U pointers of the P ranks][T pointers of the P ranks].
// Emulated: the other ranks' buffers on this device.  NCCL: CUDA IPC handles of U and T all-gathered
// over the communicator and opened (peer access over NVLink / NVSwitch).
fif_status peer_setup(DistPlan& D) {
  const int P = D.P, nl = (int)D.ranks.size();
  std::vector<void*> tab((size_t)nl * 2 * P, nullptr);
  if (D.emulated) {
    for (int li = 0; li < nl; ++li)
      for (int q = 0; q < P; ++q) {
        tab[(size_t)li * 2 * P + q] = D.ranks[q].U;
        tab[(size_t)li * 2 * P + P + q] = D.ranks[q].T;
      }
  } else {
    struct H { cudaIpcMemHandle_t u, t; };
    H mine;
    if (cudaIpcGetMemHandle(&mine.u, D.ranks[0].U) != cudaSuccess ||
        cudaIpcGetMemHandle(&mine.t, D.ranks[0].T) != cudaSuccess)
      return FIF_ERR_CUDA;
    void* dh = nullptr;
    if (cudaMalloc(&dh, sizeof(H) * (P + 1)) != cudaSuccess) return FIF_ERR_OOM;
    cudaMemcpy((char*)dh + sizeof(H) * P, &mine, sizeof(H), cudaMemcpyHostToDevice);
    fif_status st = nccl_check(nccl().allGather((char*)dh + sizeof(H) * P, dh, sizeof(H), ncclUint8, D.comm, 0),
                               "ncclAllGather(ipc handles)");
    std::vector<H> all(P);
    if (st == FIF_OK && (cudaStreamSynchronize(0) != cudaSuccess ||
                         cudaMemcpy(all.data(), dh, sizeof(H) * P, cudaMemcpyDeviceToHost) != cudaSuccess))
      st = FIF_ERR_CUDA;
    cudaFree(dh);
    if (st != FIF_OK) return st;
    for (int q = 0; q < P; ++q) {
      if (q == D.rank) {
        tab[q] = D.ranks[0].U;
        tab[P + q] = D.ranks[0].T;
        continue;
      }
      if (cudaIpcOpenMemHandle(&tab[q], all[q].u, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
          cudaIpcOpenMemHandle(&tab[P + q], all[q].t, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return FIF_ERR_CUDA;
      D.ipc_open.push_back(tab[q]);
      D.ipc_open.push_back(tab[P + q]);
    }
    if (cudaMalloc(&D.dbar, 16) != cudaSuccess) return FIF_ERR_OOM;
  }
  if (cudaMalloc(&D.dpeer, sizeof(void*) * tab.size()) != cudaSuccess) return FIF_ERR_OOM;
  if (cudaMemcpy(D.dpeer, tab.data(), sizeof(void*) * tab.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return FIF_ERR_CUDA;
  D.hpeer = tab;
  D.peer = true;
  return FIF_OK;
}
// every rank's peer stores issued so far are complete and visible (stream-ordered)
fif_status peer_barrier(DistPlan& D, cudaStream_t s) {
  if (D.emulated) return FIF_OK;  // one stream: program order
  return nccl_check(nccl().allReduce(D.dbar, D.dbar, 1, ncclInt32, ncclSum, D.comm, s), "ncclAllReduce(barrier)");
}

// The whole decomposition, phase by phase: each phase's kernels for every local rank, then the
// phase's collective.  Static schedule (every rank issues the same collectives in the same order,
// active or not).  Inverse buffers: pre -> T, local passes on T, twiddle T -> U, all-to-all U -> T,
// rank IDFT T -> U, all-to-all U -> T, epilogue T -> IMF slot M (device-resolved) and R.
template <typename Real>
fif_status dist_decompose_t(fif_plan_s* p, DistPlan& D, const void* sig, void* imfs, int32_t* cnt, int32_t* lens,
                            int32_t* its, cudaStream_t s) {
  using V = typename Cx<Real>::V;
  const Tabs<Real> tb{(const double2*)D.Eh, (const double2*)D.El, (const V*)D.Th, (const V*)D.Tl, (const V*)D.tw};
  const int nl = (int)D.ranks.size();
  const int64_t Q = D.Q, W = Q / D.P;
  const int TB = kThreads;
  const int64_t sig_stride = 2 * Q, out_stride = (int64_t)(p->max_imfs + 1) * 2 * Q;
  auto SIG = [&](int li) { return (const Real*)sig + li * sig_stride; };
  auto OUT = [&](int li) { return (Real*)imfs + li * out_stride; };
  const int ge = gmin((Q + TB - 1) / TB, D.grid_elem);
  const int gw = gmin((W + TB - 1) / TB, D.grid_elem);
  const int gp = D.grid_probe;
  const int gs = gmin((Q / 2048 + 1) * 8 / 8 + 1, D.grid_elem);
  const bool fast = p->max_inner == kFastCap;
  fif_status st = FIF_OK;
  auto ok = [&](fif_status x) { if (st == FIF_OK) st = x; };
  auto all = [&](auto fn) { for (int li = 0; li < nl; ++li) fn(li, D.ranks[li]); };
  for (DRank& R : D.ranks) {  // method options (fif_plan_set_options)
    R.d.g.stop = p->stop;
    R.d.g.delta = p->delta;
    R.d.g.gamma = p->gamma;
  }
  const size_t qb = sizeof(V) * (size_t)Q, wb = sizeof(V) * (size_t)W;
  auto ext_gather = [&]() {
    ok(c_allgather(D, [&](int, DRank& R) { return (const void*)R.c.ext_send; },
                   [&](int, DRank& R) { return (void*)R.c.ext_recv; }, sizeof(DExt), s));
  };
  auto probe_gather = [&]() {
    ok(c_allgather(D, [&](int, DRank& R) { return (const void*)R.c.pr_send; },
                   [&](int, DRank& R) { return (void*)R.c.pr_recv; }, 2 * kProbes * sizeof(double), s));
  };

  // ---- a1 input, a2/a3 extrema of s
  all([&](int li, DRank& R) {
    k_d_init<<<1, 32, 0, s>>>(R.c.s);
    k_d_load<Real><<<gs, TB, 0, s>>>(R.d, SIG(li), OUT(li) + (int64_t)p->max_imfs * 2 * Q, R.c);
    k_d_fold_local<<<1, TB, 0, s>>>(R.d, R.c, 1);
  });
  ext_gather();
  all([&](int li, DRank& R) { k_d_decide_ext<<<1, 1, 0, s>>>(R.d, R.c, 0, lens + li * p->max_imfs, its + li * p->max_imfs); });
  // ---- a1 forward transform
  Nvtx fwd_range("distributed/forward");
  // peer tables of local rank li: U pointers, T pointers (device), and the partner's T (host value)
  auto ptabU = [&](int li) { return (V* const*)((void**)D.dpeer + (size_t)li * 2 * D.P); };
  auto ptabT = [&](int li) { return (V* const*)((void**)D.dpeer + (size_t)li * 2 * D.P + D.P); };
  if (D.peer) {
    const std::vector<void*>& tab = D.hpeer;  // host copy kept by peer_setup: no device read, graph-capturable
    all([&](int li, DRank& R) { k_d_scatter<Real><<<ge, TB, 0, s>>>(R.d, (const V*)SIG(li), ptabU(li)); });
    ok(peer_barrier(D, s));
    all([&](int li, DRank& R) {
      k_d_rankdft<Real, -1><<<gw, TB, 0, s>>>(R.d, (const V*)R.U, nullptr, tb, R.c.s, ptabT(li));
    });
    ok(peer_barrier(D, s));
    all([&](int, DRank& R) {
      for (int i = 0; i < R.d.g.L; ++i)
        launch_dpass<Real, -1>(D.pass_cs[i], gmin(R.d.g.lv[i].tiles, D.grid_pass), D.smem_pass[i], s, R.d, R.d.g.lv[i],
                               (V*)R.T, tb, (const int32_t*)R.c.s);
    });
    ok(peer_barrier(D, s));
    all([&](int li, DRank& R) {
      const int pr = (D.P - R.d.rank) % D.P;
      const V* Zp = (const V*)tab[(size_t)li * 2 * D.P + D.P + pr];  // the partner's spectrum, read over NVLink
      k_d_post<Real><<<ge, TB, 0, s>>>(R.d, (const V*)R.T, Zp, (V*)R.X, (V*)R.Xm, tb, R.c.s);
    });
    ok(peer_barrier(D, s));  // the partner has read our T before our first damping overwrites it
  } else {
    ok(c_alltoall(D, [&](int li, DRank&) { return (const void*)SIG(li); }, [&](int, DRank& R) { return R.U; }, wb, s));
    all([&](int, DRank& R) { k_d_rankdft<Real, -1><<<gw, TB, 0, s>>>(R.d, (const V*)R.U, (V*)R.T, tb, R.c.s); });
    ok(c_alltoall(D, [&](int, DRank& R) { return (const void*)R.T; }, [&](int, DRank& R) { return R.U; }, wb, s));
    all([&](int, DRank& R) {
      for (int i = 0; i < R.d.g.L; ++i)
        launch_dpass<Real, -1>(D.pass_cs[i], gmin(R.d.g.lv[i].tiles, D.grid_pass), D.smem_pass[i], s, R.d, R.d.g.lv[i],
                               (V*)R.U, tb, (const int32_t*)R.c.s);
    });
    ok(c_partner(D, [&](int, DRank& R) { return (const void*)R.U; }, [&](int, DRank& R) { return R.T; }, qb, s));
    all([&](int, DRank& R) {
      k_d_post<Real><<<ge, TB, 0, s>>>(R.d, (const V*)R.U, (const V*)R.T, (V*)R.X, (V*)R.Xm, tb, R.c.s);
    });
  }
  // ---- IMFs
  for (int m = 0; m < p->max_imfs; ++m) {
    Nvtx imf_range("distributed/imf");
    // a4/a5: cap probe, then K-ary rounds (device-side early exit when not searching)
    all([&](int, DRank& R) {
      if (fast) k_d_probe<Real, kFastCap, 0><<<gp, TB, 0, s>>>(R.d, (const V*)R.X, (const V*)R.Xm, tb, R.c);
      else k_d_probe<Real, 0, 0><<<gp, TB, 0, s>>>(R.d, (const V*)R.X, (const V*)R.Xm, tb, R.c);
    });
    probe_gather();
    all([&](int, DRank& R) { k_d_decide_probe<0><<<1, 1, 0, s>>>(R.d, R.c); });
    for (int r = 0; r < D.rounds; ++r) {
      all([&](int, DRank& R) { k_d_probe<Real, 0, 1><<<gp, TB, 0, s>>>(R.d, (const V*)R.X, (const V*)R.Xm, tb, R.c); });
      probe_gather();
      all([&](int, DRank& R) { k_d_decide_probe<1><<<1, 1, 0, s>>>(R.d, R.c); });
    }
    // a6: damping + pre-processing, local inverse passes, twiddle
    all([&](int, DRank& R) {
      if (fast) k_d_pre<Real, kFastCap><<<ge, TB, 0, s>>>(R.d, (V*)R.X, (V*)R.Xm, (V*)R.T, tb, R.c.s);
      else k_d_pre<Real, 0><<<ge, TB, 0, s>>>(R.d, (V*)R.X, (V*)R.Xm, (V*)R.T, tb, R.c.s);
      for (int i = R.d.g.L - 1; i >= 0; --i)
        launch_dpass<Real, 1>(D.pass_cs[i], gmin(R.d.g.lv[i].tiles, D.grid_pass), D.smem_pass[i], s, R.d, R.d.g.lv[i],
                              (V*)R.T, tb, (const int32_t*)R.c.s);
      if (!D.peer) k_d_twiddle_inv<Real><<<ge, TB, 0, s>>>(R.d, (const V*)R.T, (V*)R.U, tb, R.c.s);
    });
    if (D.peer) {  // all-to-alls #3 and #4 as peer stores of the twiddle and rank-DFT kernels
      all([&](int li, DRank& R) { k_d_twiddle_scatter<Real><<<ge, TB, 0, s>>>(R.d, (const V*)R.T, ptabU(li), tb, R.c.s); });
      ok(peer_barrier(D, s));
      all([&](int li, DRank& R) {
        k_d_rankdft<Real, 1><<<gw, TB, 0, s>>>(R.d, (const V*)R.U, nullptr, tb, R.c.s, ptabT(li));
      });
      ok(peer_barrier(D, s));
    } else {
      ok(c_alltoall(D, [&](int, DRank& R) { return (const void*)R.U; }, [&](int, DRank& R) { return R.T; }, wb, s));
      all([&](int, DRank& R) { k_d_rankdft<Real, 1><<<gw, TB, 0, s>>>(R.d, (const V*)R.T, (V*)R.U, tb, R.c.s); });
      ok(c_alltoall(D, [&](int, DRank& R) { return (const void*)R.U; }, [&](int, DRank& R) { return R.T; }, wb, s));
    }
    all([&](int li, DRank& R) {
      k_d_epi<Real><<<ge, TB, 0, s>>>(R.d, (const V*)R.T, OUT(li), R.c);
      k_d_segs<Real><<<gs, TB, 0, s>>>(R.d, OUT(li), R.c);
      k_d_fold_local<<<1, TB, 0, s>>>(R.d, R.c, 0);
    });
    ext_gather();
    all([&](int li, DRank& R) { k_d_decide_ext<<<1, 1, 0, s>>>(R.d, R.c, 1, lens + li * p->max_imfs, its + li * p->max_imfs); });
  }
  // ---- a7
  all([&](int li, DRank& R) {
    k_d_final<Real><<<ge, TB, 0, s>>>(R.d, OUT(li), R.c.s, cnt + li, lens + li * p->max_imfs, its + li * p->max_imfs);
    k_d_zero<Real><<<ge, TB, 0, s>>>(R.d, OUT(li), R.c.s);
  });
  return st;
}

fif_status dist_setup(fif_plan_s* p, DistPlan& D) {
  return p->dtype == FIF_F64 ? dist_setup_t<double>(p, D) : dist_setup_t<float>(p, D);
}

}  // namespace

fif_status dist_create(fif_plan_s* p, const void* uid, int rank, int nranks, int emulated) {
  DistPlan* D = new DistPlan();
  p->dist = D;
  D->P = nranks;
  D->rank = emulated ? 0 : rank;
  D->emulated = emulated != 0;
  // FIF_DIST_FORCE_NCCL: a one-rank plan still goes through NCCL (self all-gathers / self send-recv),
  // which exercises the NCCL path on a single GPU (tests)
  const bool force = getenv("FIF_DIST_FORCE_NCCL") != nullptr;
  if (!D->emulated && (nranks > 1 || force)) {
    if (!nccl().load()) return FIF_ERR_NCCL;
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    fif_status st = nccl_check(nccl().commInitRank(&D->comm, nranks, id, rank), "ncclCommInitRank");
    if (st != FIF_OK) return st;
  } else if (!D->emulated) {
    D->emulated = true;  // a one-rank "distributed" plan needs no communicator
  }
  fif_status st = dist_setup(p, *D);
  if (st == FIF_OK && getenv("FIF_DIST_PEER")) st = peer_setup(*D);
  return st;
}
fif_status dist_decompose(fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its,
                          cudaStream_t s) {
  DistPlan& D = *p->dist;
  // NCCL failures of earlier (asynchronous) calls surface here: a communicator in error refuses new work
  if (fif_status a = async_error(D); a != FIF_OK) return a;
  const fif_status st = p->dtype == FIF_F64 ? dist_decompose_t<double>(p, D, sig, imfs, cnt, lens, its, s)
                                            : dist_decompose_t<float>(p, D, sig, imfs, cnt, lens, its, s);
  if (st != FIF_OK) return st;
  return async_error(D);
}
void dist_free(fif_plan_s* p) {
  DistPlan* D = p->dist;
  if (!D) return;
  for (DRank& R : D->ranks) {
    cudaFree(R.X);
    cudaFree(R.Xm);
    cudaFree(R.T);
    cudaFree(R.U);
    cudaFree(R.small);
  }
  cudaFree(D->Eh);
  cudaFree(D->El);
  cudaFree(D->Th);
  cudaFree(D->Tl);
  cudaFree(D->tw);
  cudaFree(D->utab);
  cudaFree(D->rbase);
  cudaFree(D->rmir);
  for (void* q : D->ipc_open) cudaIpcCloseMemHandle(q);
  cudaFree(D->dpeer);
  cudaFree(D->dbar);
  if (D->comm) nccl().commDestroy(D->comm);
  delete D;
  p->dist = nullptr;
}
int dist_kernels_per_call(const fif_plan_s* p) {
  const DistPlan& D = *p->dist;
  const int L = D.ranks.empty() ? 0 : D.ranks[0].d.g.L;
  const int per_rank = 4 + 2 + L + 1 + p->max_imfs * (2 + 2 * D.rounds + 1 + L + 1 + 1 + 3 + 1) + 2;
  return per_rank * (int)D.ranks.size();
}
fif_status nccl_unique_id(void* out) {
  if (!nccl().load()) return FIF_ERR_NCCL;
  ncclUniqueId id;
  fif_status st = nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
  if (st == FIF_OK) memcpy(out, &id, sizeof(id));
  return st;
}

}  // namespace fifhost
