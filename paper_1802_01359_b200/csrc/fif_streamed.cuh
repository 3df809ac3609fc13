// fif_streamed.cuh -- the "streamed" regime of the FIF hot path for n beyond on-chip capacity
// (configs 2 and 4: n up to 2^22, radix 2/3/4/5/8).  The spectrum X (transposed four-step order), an
// FFT work buffer Z and the time-domain remainder R live in HBM; every IMF is a fixed sequence of
// stream-ordered kernels over the whole batch, with per-signal state (k, L, N, M, done) in device
// arrays so that no host round trip happens inside fif_decompose.
//
// Same method and readings as fif_resident.cuh:
//   a1  forward four-step FFT of z_m = s_2m + i s_2m+1 (columns, then rows; output in transposed
//       order: position k1 N2 + k2 holds bin k1 + N1 k2) + Hermitian post-processing
//   a2  extrema monoid per chunk of R, ordered fold per signal (reading A4)
//   a3  L from k (A1, A3, A8)
//   a4  w_hat_k = [sin(pi r/n) / (L sin(pi k/n))]^4 with exact integer reduction, sinpi
//   a5  fp64 cap probe, then K-ary fp64 search passes when SD(cap) <= delta (monotone SD)
//   a6  damping + pre-processing, inverse four-step (rows, then columns -> natural order),
//       IMF store and R -= IMF in the last kernel's epilogue
//   a7  counts, trend in slot M, zero fill
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fif_resident.cuh"

namespace fifgpu {
namespace st {

constexpr int kMaxPass = 16;
constexpr int kProbes = 15;  // K-ary search: probes per pass
constexpr int kThreads = 256;

struct Geo {
  int64_t n, NC, batch;
  int N1, N2;                      // NC = N1 * N2
  int C;                           // columns per CTA in the column kernels
  int rad1[kMaxPass], np1;         // radix schedule of the N1-point FFTs
  int rad2[kMaxPass], np2;         // radix schedule of the N2-point FFTs
  int binch, nbch;                 // bins per chunk (reductions), chunks per signal
  int smpch, nsch;                 // samples per extrema chunk, chunks per signal
  int max_imfs, max_inner, window;
  double xi, delta2;
};

// per-signal control block (device)
struct Ctl {
  int32_t* k;       // extrema count of the current remainder
  int32_t* L;       // half-length of h for the current IMF
  int32_t* N;       // iteration count of the current IMF
  int32_t* M;       // IMFs done
  int32_t* active;  // 1 while the current IMF is being extracted
  int32_t* search;  // 1 while the K-ary search runs
  int32_t* lo;      // search bracket: !pass(lo) (lo = 0 virtual), pass(hi)
  int32_t* hi;
  int32_t* bad;     // non-finite input
  int32_t* ext;     // [B][nsch][3] extrema partials (first sign, last sign, changes)
  double* red;      // [B][nbch][2*kProbes] reduction partials
};

// ------------------------------------------------------------------ small DFTs (radix 2, 3, 4, 5, 8)
template <int DIR, typename V>
__device__ __forceinline__ void dft3(V& x0, V& x1, V& x2) {
  using S = decltype(x0.x);
  const S h = (S)0.86602540378443864676372317075293618;  // sqrt(3)/2
  const V t = cadd(x1, x2);
  const V u = mul_i<DIR>(cscale(csub(x1, x2), h));
  const V m = V{x0.x - (S)0.5 * t.x, x0.y - (S)0.5 * t.y};
  x0 = cadd(x0, t);
  x1 = cadd(m, u);
  x2 = csub(m, u);
}
template <int DIR, typename V>
__device__ __forceinline__ void dft5(V& x0, V& x1, V& x2, V& x3, V& x4) {
  using S = decltype(x0.x);
  const S c1 = (S)0.30901699437494742410229341718281906, c2 = (S)-0.80901699437494742410229341718281906;
  const S s1 = (S)0.95105651629515357211643933337938214, s2 = (S)0.58778525229247312916870595463907277;
  const V a1 = cadd(x1, x4), a2 = cadd(x2, x3), b1 = csub(x1, x4), b2 = csub(x2, x3);
  const V t1 = V{x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y};
  const V t2 = V{x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y};
  const V u1 = mul_i<DIR>(V{s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y});
  const V u2 = mul_i<DIR>(V{s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y});
  x0 = cadd(x0, cadd(a1, a2));
  x1 = cadd(t1, u1);
  x4 = csub(t1, u1);
  x2 = cadd(t2, u2);
  x3 = csub(t2, u2);
}

// One Stockham pass of radix p (runtime) over F independent FFTs of length Ns stored contiguously:
// src[f*Ns + i] -> dst[f*Ns + j].  tw[j] = e^{-2 pi i j/Ns}.
template <int DIR, typename V>
__device__ void cta_pass(const V* src, V* dst, int Ns, int F, int p, int NS, const V* __restrict__ tw) {
  const int per = Ns / p;
  const int tstride = Ns / (NS * p);
  for (int idx = threadIdx.x; idx < F * per; idx += blockDim.x) {
    const int f = idx / per, vt = idx - f * per;
    const int k = vt % NS;
    const V* s = src + (size_t)f * Ns + vt;
    V x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (r < p) x[r] = s[r * per];
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < 8; ++r)
        if (r < p) {
          V t = __ldg(tw + (size_t)k * r * tstride);
          if (DIR > 0) t.y = -t.y;
          x[r] = cmul(x[r], t);
        }
    }
    switch (p) {
      case 2: { V a = cadd(x[0], x[1]), b = csub(x[0], x[1]); x[0] = a; x[1] = b; } break;
      case 3: dft3<DIR>(x[0], x[1], x[2]); break;
      case 4: dft4<DIR>(x[0], x[1], x[2], x[3]); break;
      case 5: dft5<DIR>(x[0], x[1], x[2], x[3], x[4]); break;
      default: dft8<DIR>(x); break;
    }
    V* d = dst + (size_t)f * Ns + (vt / NS) * NS * p + k;
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (r < p) d[r * NS] = x[r];
  }
}

// All passes; a holds the input, returns the buffer holding the output (a or b).
template <int DIR, typename V>
__device__ V* cta_fft(V* a, V* b, int Ns, int F, const int* rad, int np, const V* __restrict__ tw) {
  int NS = 1;
  for (int ps = 0; ps < np; ++ps) {
    __syncthreads();
    cta_pass<DIR>(a, b, Ns, F, rad[ps], NS, tw);
    NS *= rad[ps];
    V* t = a; a = b; b = t;
  }
  __syncthreads();
  return a;
}

// e^{s 2 pi i m / Nmod} with exact integer reduction of m (sincospi argument 2 m / Nmod)
template <typename V>
__device__ __forceinline__ V cis(int64_t m, int64_t Nmod, int sgn) {
  m %= Nmod;
  if (m < 0) m += Nmod;
  double s, c;
  sincospi(2.0 * (double)m / (double)Nmod, &s, &c);
  using S = decltype(V{}.x);
  return V{(S)c, (S)(sgn * s)};
}

// ------------------------------------------------------------------ window spectrum (a4)
__device__ __forceinline__ double what_st(int64_t n, int L, int64_t k) {
  if (k == 0) return 1.0;
  int64_t m = ((int64_t)L * k) % n;
  const int64_t r = m < n - m ? m : n - m;
  const int64_t kk = k < n - k ? k : n - k;
  const double s = sinpi((double)r / (double)n) / ((double)L * sinpi((double)kk / (double)n));
  const double s2 = s * s;
  return s2 * s2;
}
__device__ __forceinline__ double upow_rt(double a, int e) {
  double r = 1.0, b = a;
  while (e) {
    if (e & 1) r *= b;
    e >>= 1;
    if (e) b *= b;
  }
  return r;
}

// transposed-order position <-> bin
__device__ __forceinline__ int64_t bin_of_pos(const Geo& g, int64_t p) {
  const int64_t k1 = p / g.N2, k2 = p - k1 * g.N2;
  return k1 + (int64_t)g.N1 * k2;
}
__device__ __forceinline__ int64_t pos_of_bin(const Geo& g, int64_t k) {
  const int64_t k1 = k % g.N1, k2 = k / g.N1;
  return k1 * g.N2 + k2;
}

// ------------------------------------------------------------------ forward a1: columns
// z = s viewed as complex [B][NC]; Z[k1 N2 + m2] = twiddle * DFT_N1 over m1 of z[N2 m1 + m2].
// Also copies s into R and flags non-finite samples.
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_fwd_cols(Geo g, const Real* __restrict__ s, Real* __restrict__ R,
                                                       typename Cx<Real>::V* __restrict__ Z,
                                                       const typename Cx<Real>::V* __restrict__ tw1, Ctl c,
                                                       int64_t R_stride) {
  using V = typename Cx<Real>::V;
  extern __shared__ __align__(16) char smem_raw[];
  V* A = reinterpret_cast<V*>(smem_raw);
  V* Bf = A + (size_t)g.N1 * g.C;
  const int64_t tiles = g.N2 / g.C;
  for (int64_t t = blockIdx.x; t < g.batch * tiles; t += gridDim.x) {
    const int64_t b = t / tiles, c0 = (t - b * tiles) * g.C;
    const V* zb = reinterpret_cast<const V*>(s + b * g.n);
    V* Rb = reinterpret_cast<V*>(R + b * R_stride);
    bool finite = true;
    // load tile (column-major in smem: column c occupies A[c*N1 .. c*N1+N1))
    for (int i = threadIdx.x; i < g.N1 * g.C; i += blockDim.x) {
      const int m1 = i / g.C, cc = i - m1 * g.C;
      const int64_t gi = (int64_t)g.N2 * m1 + c0 + cc;
      const V v = zb[gi];
      finite &= isfinite(v.x) && isfinite(v.y);
      Rb[gi] = v;
      A[cc * g.N1 + m1] = v;
    }
    if (!finite) atomicOr(c.bad + b, 1);
    V* out = cta_fft<-1>(A, Bf, g.N1, g.C, g.rad1, g.np1, tw1);
    V* Zb = Z + b * g.NC;
    for (int i = threadIdx.x; i < g.N1 * g.C; i += blockDim.x) {
      const int k1 = i / g.C, cc = i - k1 * g.C;
      const int64_t m2 = c0 + cc;
      V v = out[cc * g.N1 + k1];
      v = cmul(v, cis<V>(m2 * k1, g.NC, -1));
      Zb[(int64_t)k1 * g.N2 + m2] = v;
    }
    __syncthreads();
  }
}

// rows: for every row of N2 contiguous elements: DFT (DIR); for DIR = +1 (inverse step B') also
// multiply by e^{+2 pi i m2 k1/NC}.  Only active signals (if only_active).
template <typename Real, int DIR>
__global__ void __launch_bounds__(kThreads) k_rows(Geo g, typename Cx<Real>::V* __restrict__ Z,
                                                   const typename Cx<Real>::V* __restrict__ tw2, Ctl c,
                                                   int only_active) {
  using V = typename Cx<Real>::V;
  extern __shared__ __align__(16) char smem_raw[];
  V* A = reinterpret_cast<V*>(smem_raw);
  V* Bf = A + g.N2;
  for (int64_t t = blockIdx.x; t < g.batch * g.N1; t += gridDim.x) {
    const int64_t b = t / g.N1;
    const int k1 = (int)(t - b * g.N1);
    if (only_active && !c.active[b]) continue;
    V* row = Z + b * g.NC + (int64_t)k1 * g.N2;
    for (int i = threadIdx.x; i < g.N2; i += blockDim.x) A[i] = row[i];
    V* out = cta_fft<DIR>(A, Bf, g.N2, 1, g.rad2, g.np2, tw2);
    for (int i = threadIdx.x; i < g.N2; i += blockDim.x) {
      V v = out[i];
      if (DIR > 0) v = cmul(v, cis<V>((int64_t)i * k1, g.NC, +1));
      row[i] = v;
    }
    __syncthreads();
  }
}

// forward post-processing: X_k = E + e^{-2 pi i k/n} O from Z_k, Z_{NC-k} (transposed positions);
// Nyquist X_NC = Re Z_0 - Im Z_0 to Xn[b].
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_fwd_post(Geo g, const typename Cx<Real>::V* __restrict__ Z,
                                                       typename Cx<Real>::V* __restrict__ X,
                                                       typename Cx<Real>::V* __restrict__ Xn) {
  using V = typename Cx<Real>::V;
  const int64_t tot = g.batch * g.NC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / g.NC, p = i - b * g.NC;
    const int64_t k = bin_of_pos(g, p);
    const V* Zb = Z + b * g.NC;
    const V P = Zb[p];
    const V Q = Zb[pos_of_bin(g, k == 0 ? 0 : g.NC - k)];
    const Real h = (Real)0.5;
    const V E = V{h * (P.x + Q.x), h * (P.y - Q.y)};
    const V D = V{h * (P.x - Q.x), h * (P.y + Q.y)};
    const V O = V{D.y, -D.x};
    V x = cadd(E, cmul(cis<V>(k, g.n, -1), O));
    if (k == 0) {
      x = V{P.x + P.y, (Real)0};
      Xn[b] = V{P.x - P.y, (Real)0};
    }
    X[b * g.NC + p] = x;
  }
}

// ------------------------------------------------------------------ a2 extrema partials
// chunk c of signal b covers differences D_i = R[i+1]-R[i] for i in [c*smpch, min((c+1)*smpch, n-1))
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_ext(Geo g, const Real* __restrict__ R, int64_t R_stride, Ctl c,
                                                  int first) {
  __shared__ int sf[kThreads], sl[kThreads], sc[kThreads];
  for (int64_t t = blockIdx.x; t < g.batch * g.nsch; t += gridDim.x) {
    const int64_t b = t / g.nsch;
    const int ch = (int)(t - b * g.nsch);
    if (!first && !c.active[b]) continue;
    const Real* Rb = R + b * R_stride;
    const int64_t i0 = (int64_t)ch * g.smpch;
    const int64_t i1 = min((int64_t)(ch + 1) * g.smpch, g.n - 1);
    // each thread folds a contiguous sub-range
    const int64_t len = i1 - i0, per = (len + blockDim.x - 1) / blockDim.x;
    const int64_t a0 = i0 + threadIdx.x * per, a1 = min(a0 + per, i1);
    int f = 0, l = 0, cnt = 0;
    if (a0 < a1) {
      Real prev = Rb[a0];
      for (int64_t i = a0; i < a1; ++i) {
        const Real x = Rb[i + 1];
        const Real d = x - prev;
        prev = x;
        if (d == (Real)0) continue;
        const int sg = d > (Real)0 ? 1 : -1;
        if (f == 0) f = sg;
        if (l != 0 && sg != l) ++cnt;
        l = sg;
      }
    }
    sf[threadIdx.x] = f; sl[threadIdx.x] = l; sc[threadIdx.x] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      int F = 0, Ls = 0, C = 0;
      for (int u = 0; u < (int)blockDim.x; ++u) {
        const int f2 = sf[u], l2 = sl[u], c2 = sc[u];
        C += c2 + ((Ls != 0 && f2 != 0 && Ls != f2) ? 1 : 0);
        if (F == 0) F = f2;
        if (l2 != 0) Ls = l2;
      }
      int32_t* e = c.ext + (b * g.nsch + ch) * 3;
      e[0] = F; e[1] = Ls; e[2] = C;
    }
    __syncthreads();
  }
}

// per-signal control: fold extrema partials -> k; decide stop / L
__global__ void k_ctl_ext(Geo g, Ctl c, int first) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < g.batch; b += (int64_t)gridDim.x * blockDim.x) {
    if (first) {
      c.M[b] = 0;
      c.active[b] = c.bad[b] ? 0 : 1;
      if (c.bad[b]) c.M[b] = -1;
    }
    if (!c.active[b]) continue;
    int F = 0, Ls = 0, C = 0;
    for (int ch = 0; ch < g.nsch; ++ch) {
      const int32_t* e = c.ext + (b * g.nsch + ch) * 3;
      C += e[2] + ((Ls != 0 && e[0] != 0 && Ls != e[0]) ? 1 : 0);
      if (F == 0) F = e[0];
      if (e[1] != 0) Ls = e[1];
    }
    c.k[b] = C;
    if (C < 2 || c.M[b] >= g.max_imfs) {
      c.active[b] = 0;
      continue;
    }
    const double tq = __dmul_rn(g.xi, (double)g.n);
    const double u = __ddiv_rn(tq, (double)C);
    long long q = (long long)floor(u);
    long long L = g.window ? 2 * q : q;
    const long long Lmax = (g.n - 1) / 4;
    if (L < 2) L = 2;
    if (L > Lmax) L = Lmax;
    c.L[b] = (int)L;
    c.search[b] = 0;
  }
}

// ------------------------------------------------------------------ a5 probes
// mode 0: cap probe (P, Q at N = max_inner); mode 1: K-ary probes N_i = lo + i*step, i = 1..kProbes
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_probe(Geo g, const typename Cx<Real>::V* __restrict__ X,
                                                    const typename Cx<Real>::V* __restrict__ Xn, Ctl c, int mode) {
  using V = typename Cx<Real>::V;
  __shared__ double sred[kThreads / 32][2 * kProbes];
  for (int64_t t = blockIdx.x; t < g.batch * g.nbch; t += gridDim.x) {
    const int64_t b = t / g.nbch;
    const int ch = (int)(t - b * g.nbch);
    if (!c.active[b] || (mode == 1 && !c.search[b])) continue;
    const int L = c.L[b];
    int N0, step, nprobe;
    if (mode == 0) { N0 = g.max_inner; step = 0; nprobe = 1; }
    else {
      const int lo = c.lo[b], hi = c.hi[b];
      step = (hi - lo + kProbes) / (kProbes + 1);
      if (step < 1) step = 1;
      N0 = lo + step;
      nprobe = kProbes;
    }
    double acc[2 * kProbes];
#pragma unroll
    for (int i = 0; i < 2 * kProbes; ++i) acc[i] = 0.0;
    const int64_t p0 = (int64_t)ch * g.binch, p1 = min(p0 + g.binch, g.NC);
    for (int64_t p = p0 + threadIdx.x; p < p1 + (ch == 0 ? 1 : 0); p += blockDim.x) {
      int64_t k;
      V x;
      double cw;
      if (p == p1) { k = g.NC; x = Xn[b]; cw = 1.0; }  // Nyquist (chunk 0 only)
      else { k = bin_of_pos(g, p); x = X[b * g.NC + p]; cw = (k == 0) ? 1.0 : 2.0; }
      const double w = what_st(g.n, L, k);
      const double a = 1.0 - w;
      const double pk = cw * ((double)x.x * (double)x.x + (double)x.y * (double)x.y);
      const double pw = pk * w * w;
      if (mode == 0) {
        const double e = upow_rt(a, N0 - 1);
        const double xx = e * e;
        acc[0] += pk * xx;
        acc[1] += pw * xx;
      } else {
        const double a2 = a * a;
        double y = upow_rt(a2, N0 - 1);
        const double z = upow_rt(a2, step);
#pragma unroll
        for (int i = 0; i < kProbes; ++i) {
          acc[2 * i] += pk * y;
          acc[2 * i + 1] += pw * y;
          y *= z;
        }
      }
    }
    const int nv = 2 * nprobe;
    for (int i = 0; i < 2 * kProbes; ++i) {
      if (i >= nv) break;
      double v = acc[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5][i] = v;
    }
    __syncthreads();
    if (threadIdx.x < nv) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += sred[w][threadIdx.x];
      c.red[(b * g.nbch + ch) * (2 * kProbes) + threadIdx.x] = v;
    }
    __syncthreads();
  }
}

// per-signal: fold probe partials (fixed order) and update N / the search bracket
__global__ void k_ctl_probe(Geo g, Ctl c, int mode) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < g.batch; b += (int64_t)gridDim.x * blockDim.x) {
    if (!c.active[b]) continue;
    if (mode == 0) {
      double P = 0.0, Q = 0.0;
      for (int ch = 0; ch < g.nbch; ++ch) {
        P += c.red[(b * g.nbch + ch) * (2 * kProbes) + 0];
        Q += c.red[(b * g.nbch + ch) * (2 * kProbes) + 1];
      }
      c.N[b] = g.max_inner;
      if (Q <= g.delta2 * P) {  // SD(cap) <= delta: search [1, cap)
        c.lo[b] = 0;
        c.hi[b] = g.max_inner;
        c.search[b] = g.max_inner > 1 ? 1 : 0;
        if (g.max_inner == 1) c.N[b] = 1;
      }
    } else {
      if (!c.search[b]) continue;
      const int lo = c.lo[b], hi = c.hi[b];
      int step = (hi - lo + kProbes) / (kProbes + 1);
      if (step < 1) step = 1;
      int nlo = lo, nhi = hi;
      for (int i = 0; i < kProbes; ++i) {
        const int Ni = lo + step * (i + 1);
        if (Ni >= hi) break;
        double P = 0.0, Q = 0.0;
        for (int ch = 0; ch < g.nbch; ++ch) {
          P += c.red[(b * g.nbch + ch) * (2 * kProbes) + 2 * i];
          Q += c.red[(b * g.nbch + ch) * (2 * kProbes) + 2 * i + 1];
        }
        if (Q <= g.delta2 * P) { nhi = Ni; break; }
        nlo = Ni;
      }
      c.lo[b] = nlo;
      c.hi[b] = nhi;
      if (nhi - nlo <= 1) {
        c.search[b] = 0;
        c.N[b] = nhi;
      }
    }
  }
}

// ------------------------------------------------------------------ a6 damping + pre-processing
// One thread per Hermitian pair (k, NC - k) (threads whose bin k > NC/2 idle; k = 0 pairs with the
// Nyquist bin): d = a^N, X <- (1 - d) X for both, and with A = d_k X_k / n, B = d_{NC-k} X_{NC-k} / n,
// Z_k = S + T, Z_{NC-k} = conj(S - T), S = A + B*, T = i e^{2 pi i k/n} (A - B*).
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_damp_pre(Geo g, typename Cx<Real>::V* __restrict__ X,
                                                       typename Cx<Real>::V* __restrict__ Xn,
                                                       typename Cx<Real>::V* __restrict__ Z, Ctl c) {
  using V = typename Cx<Real>::V;
  const int64_t tot = g.batch * g.NC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / g.NC, p = i - b * g.NC;
    const int64_t k = bin_of_pos(g, p);
    if (2 * k > g.NC) continue;  // handled by the mirror bin's thread
    if (!c.active[b]) continue;
    const int L = c.L[b], N = c.N[b];
    const int64_t km = g.NC - k;  // == NC (Nyquist) for k = 0
    const int64_t pm = (k == 0) ? -1 : pos_of_bin(g, km);
    V* Xb = X + b * g.NC;
    const V xk = Xb[p];
    const V xm = (k == 0) ? Xn[b] : Xb[pm];
    const double dk = upow_rt(1.0 - what_st(g.n, L, k), N);
    const double dm = upow_rt(1.0 - what_st(g.n, L, km), N);
    const Real invn = (Real)(1.0 / (double)g.n);
    const V A = cscale(xk, (Real)dk * invn), B = cscale(xm, (Real)dm * invn);
    const V S = V{A.x + B.x, A.y - B.y};
    const V D = V{A.x - B.x, A.y + B.y};
    const V Tm = mul_i<1>(cmul(cis<V>(k, g.n, +1), D));
    V* Zb = Z + b * g.NC;
    Zb[p] = cadd(S, Tm);
    Xb[p] = cscale(xk, (Real)(1.0 - dk));
    if (k == 0) {
      Xn[b] = cscale(xm, (Real)(1.0 - dm));
    } else if (km != k) {
      Zb[pm] = cconj(csub(S, Tm));
      Xb[pm] = cscale(xm, (Real)(1.0 - dm));
    }
  }
}

// inverse columns (step A'): DFT(+1) over k1 of column m2 -> natural-order z[N2 m1 + m2];
// epilogue: IMF pair (Re, Im) -> imfs slot M, R -= IMF.
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_inv_cols(Geo g, const typename Cx<Real>::V* __restrict__ Z,
                                                       const typename Cx<Real>::V* __restrict__ tw1,
                                                       Real* __restrict__ imfs, Real* __restrict__ R,
                                                       int64_t sig_stride, Ctl c) {
  using V = typename Cx<Real>::V;
  extern __shared__ __align__(16) char smem_raw[];
  V* A = reinterpret_cast<V*>(smem_raw);
  V* Bf = A + (size_t)g.N1 * g.C;
  const int64_t tiles = g.N2 / g.C;
  for (int64_t t = blockIdx.x; t < g.batch * tiles; t += gridDim.x) {
    const int64_t b = t / tiles, c0 = (t - b * tiles) * g.C;
    if (!c.active[b]) continue;
    const V* Zb = Z + b * g.NC;
    for (int i = threadIdx.x; i < g.N1 * g.C; i += blockDim.x) {
      const int k1 = i / g.C, cc = i - k1 * g.C;
      A[cc * g.N1 + k1] = Zb[(int64_t)k1 * g.N2 + c0 + cc];
    }
    V* out = cta_fft<1>(A, Bf, g.N1, g.C, g.rad1, g.np1, tw1);
    V* imf = reinterpret_cast<V*>(imfs + b * sig_stride + (int64_t)c.M[b] * g.n);
    V* Rb = reinterpret_cast<V*>(R + b * sig_stride);
    for (int i = threadIdx.x; i < g.N1 * g.C; i += blockDim.x) {
      const int m1 = i / g.C, cc = i - m1 * g.C;
      const int64_t m = (int64_t)g.N2 * m1 + c0 + cc;
      const V v = out[cc * g.N1 + m1];
      __stcs(imf + m, v);
      Rb[m] = csub(Rb[m], v);
    }
    __syncthreads();
  }
}

// per-signal bookkeeping after an IMF
__global__ void k_ctl_done(Geo g, Ctl c, int32_t* lens, int32_t* iters) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < g.batch; b += (int64_t)gridDim.x * blockDim.x) {
    if (!c.active[b]) continue;
    const int M = c.M[b];
    lens[b * g.max_imfs + M] = 2 * c.L[b];
    iters[b * g.max_imfs + M] = c.N[b];
    c.M[b] = M + 1;
  }
}

// final: trend (R lives in slot max_imfs) to slot M, zeros after; counts; zero lens/iters past M
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_final(Geo g, Real* __restrict__ imfs, int64_t sig_stride, Ctl c,
                                                    int32_t* count, int32_t* lens, int32_t* iters) {
  for (int64_t t = blockIdx.x; t < g.batch; t += gridDim.x) {
    const int M = c.M[t];
    Real* base = imfs + t * sig_stride;
    const Real* R = base + (int64_t)g.max_imfs * g.n;
    if (M < 0) {  // non-finite input
      for (int64_t i = threadIdx.x; i < (int64_t)(g.max_imfs + 1) * g.n; i += blockDim.x) base[i] = (Real)0;
    } else if (M < g.max_imfs) {
      Real* tr = base + (int64_t)M * g.n;
      for (int64_t i = threadIdx.x; i < g.n; i += blockDim.x) tr[i] = R[i];
      __syncthreads();
      for (int64_t i = (int64_t)(M + 1) * g.n + threadIdx.x; i < (int64_t)(g.max_imfs + 1) * g.n; i += blockDim.x)
        base[i] = (Real)0;
    }
    for (int m = threadIdx.x; m < g.max_imfs; m += blockDim.x)
      if (m >= M) { lens[t * g.max_imfs + m] = 0; iters[t * g.max_imfs + m] = 0; }
    if (threadIdx.x == 0) count[t] = M;
    __syncthreads();
  }
}

}  // namespace st
}  // namespace fifgpu
