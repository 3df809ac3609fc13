// fif_resident.cuh -- the on-chip-resident FIF kernel for sm_100a.
//
// One CTA decomposes one signal at a time (persistent over the batch): the
// remainder r (time domain) and its spectrum r_hat stay in REGISTERS for all
// IMFs; shared memory holds only the FFT exchange buffers and the sin table.
// HBM traffic per signal is the compulsory one: read s once, write every IMF
// and the trend once.
//
// Steps (PAPER.md passages):
//   a1  forward rfft of s, once           ("U^T s is the DFT of s")
//   a2  extrema count k of r              (reading A4)
//   a3  L = clamp(floor(fl(fl(xi n)/k)))  (A1, A3, A8)
//   a4  w_hat_k = [sin(pi r_k/n) / (L sin(pi k/n))]^4 with exact integer
//       reduction r_k = min(Lk mod n, n - Lk mod n)   (closed form of DFT(h(*)h),
//       PAPER.md:543 eigenvalues = DFT of the filter row; DESIGN.md derivation)
//   a5  N = min{N : Q(N) <= delta^2 P(N)}, cap first then bisection
//       (Parseval :175-180; monotone SD, P7)
//   a6  IMF = IRFFT(a^N r_hat), r_hat <- r_hat (1 - a^N), r <- r - IMF
//       (PAPER.md:688 Eq. One step_algo; :344 s_hat_2 = [1-(1-w_hat)^N] s_hat; :413)
//   a7  outer loop control, trend, zero fill
//
// FFT: n real points = NC = n/2 complex points (z_m = x_2m + i x_2m+1), Stockham
// auto-sort passes (radix 8, plus one radix-2/4 first pass), each thread owning
// R = 8 complex values at positions j + T*q.  The first forward pass reads from
// registers and the last pass of either direction ends in registers, so the
// time-domain data never round-trips through shared memory at the ends.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef FIF_MINB
#define FIF_MINB 2
#endif

namespace fifgpu {

// ------------------------------------------------------------------ types
template <typename Real> struct Cx;
template <> struct Cx<double> { using V = double2; };
template <> struct Cx<float> { using V = float2; };

struct Params {
  int64_t batch;
  double xi;
  double delta2;    // delta^2 (stopping test Q <= delta^2 P)
  int32_t max_inner;
  int32_t max_imfs;
  int32_t window;   // 0 = R1, 1 = R3 (wide)
};

// ------------------------------------------------------------------ radix schedule (compile time)
__host__ __device__ constexpr int sched_r0(int NC, int R) {
  int m = NC;
  while (m % R == 0 && m > 1) m /= R;
  return m;  // leftover factor (1, 2 or 4 for power-of-two NC and R = 8)
}
__host__ __device__ constexpr int sched_passes(int NC, int R) {
  int m = NC, p = 0;
  while (m % R == 0 && m > 1) { m /= R; ++p; }
  return p + (m > 1 ? 1 : 0);
}
__host__ __device__ constexpr int sched_radix(int NC, int R, int p) {
  return (sched_r0(NC, R) > 1 && p == 0) ? sched_r0(NC, R) : R;
}
__host__ __device__ constexpr int sched_ns(int NC, int R, int p) {
  int ns = 1;
  for (int i = 0; i < p; ++i) ns *= sched_radix(NC, R, i);
  return ns;
}
// offset (in complex elements) of pass p's twiddle block tw[(r-1)*NS + k], r = 1..RP-1, k < NS
__host__ __device__ constexpr int sched_twoff(int NC, int R, int p) {
  int off = 0;
  for (int i = 1; i < p; ++i) off += (sched_radix(NC, R, i) - 1) * sched_ns(NC, R, i);
  return off;
}
__host__ __device__ constexpr int sched_twtotal(int NC, int R) { return sched_twoff(NC, R, sched_passes(NC, R)); }

// ------------------------------------------------------------------ complex helpers
template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return V{a.x + b.x, a.y + b.y}; }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return V{a.x - b.x, a.y - b.y}; }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  return V{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename V> __device__ __forceinline__ V cconj(V a) { return V{a.x, -a.y}; }
// multiply by DIR * i
template <int DIR, typename V> __device__ __forceinline__ V mul_i(V a) {
  return DIR > 0 ? V{-a.y, a.x} : V{a.y, -a.x};
}

// In-place radix-RP DFTs, X_k = sum_j v_j e^{DIR 2 pi i jk/RP}, natural order in and out.
template <int DIR, typename V> __device__ __forceinline__ void dft4(V& v0, V& v1, V& v2, V& v3) {
  V b0 = cadd(v0, v2), b1 = csub(v0, v2), b2 = cadd(v1, v3), b3 = mul_i<DIR>(csub(v1, v3));
  v0 = cadd(b0, b2); v2 = csub(b0, b2); v1 = cadd(b1, b3); v3 = csub(b1, b3);
}

template <int DIR, typename V> __device__ __forceinline__ void dft8(V* v) {
  using S = decltype(v[0].x);
  const S c = (S)0.70710678118654752440084436210484903928;
  V u0 = cadd(v[0], v[4]), u1 = cadd(v[1], v[5]), u2 = cadd(v[2], v[6]), u3 = cadd(v[3], v[7]);
  V t0 = csub(v[0], v[4]), t1 = csub(v[1], v[5]), t2 = csub(v[2], v[6]), t3 = csub(v[3], v[7]);
  // t_j *= w^j, w = e^{DIR i pi/4}
  t1 = V{c * (t1.x - (S)DIR * t1.y), c * ((S)DIR * t1.x + t1.y)};
  t2 = mul_i<DIR>(t2);
  t3 = V{c * (-t3.x - (S)DIR * t3.y), c * ((S)DIR * t3.x - t3.y)};
  dft4<DIR>(u0, u1, u2, u3);
  dft4<DIR>(t0, t1, t2, t3);
  v[0] = u0; v[1] = t0; v[2] = u1; v[3] = t1; v[4] = u2; v[5] = t2; v[6] = u3; v[7] = t3;
}

template <int RP, int DIR, typename V> struct Dft;
template <int DIR, typename V> struct Dft<2, DIR, V> {
  __device__ __forceinline__ static void run(V* v) { V a = cadd(v[0], v[1]), b = csub(v[0], v[1]); v[0] = a; v[1] = b; }
};
template <int DIR, typename V> struct Dft<4, DIR, V> {
  __device__ __forceinline__ static void run(V* v) { dft4<DIR>(v[0], v[1], v[2], v[3]); }
};
template <int DIR, typename V> struct Dft<8, DIR, V> {
  __device__ __forceinline__ static void run(V* v) { dft8<DIR>(v); }
};

// shared-memory padding: one pad element per 128 bytes of data (bank-conflict-free
// strided Stockham stores)
template <typename V> __device__ __forceinline__ int pad(int i) {
  return sizeof(V) == 16 ? i + (i >> 3) : i + (i >> 4);
}
template <typename V> __host__ __device__ constexpr int padded_len(int n) {
  return sizeof(V) == 16 ? n + (n >> 3) + 1 : n + (n >> 4) + 1;
}

// ------------------------------------------------------------------ one Stockham pass
// Virtual threads vt in [0, NC/RP): inputs x[vt + r NC/RP], twiddle e^{DIR 2 pi i k r/(NS RP)}
// with k = vt mod NS, radix-RP DFT, outputs y[(vt/NS) NS RP + k + r NS].
// Real thread j runs virtual threads vt = j + T u, u < R/RP; its register q = u + r (R/RP)
// holds position j + T q, which is exactly vt + r NC/RP.
template <typename V, int NC, int R, int RP, int NS, int DIR, bool FROM_REGS, bool TO_REGS>
__device__ __forceinline__ void stockham_pass(V (&v)[R], const V* src, V* dst, const V* __restrict__ tw, int j) {
  constexpr int T = NC / R, VP = R / RP;
  if (!FROM_REGS) {
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = src[pad<V>(j + T * q)];
  }
#pragma unroll
  for (int u = 0; u < VP; ++u) {
    const int vt = j + T * u;
    const int k = vt & (NS - 1);
    V w[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) w[r] = v[u + r * VP];
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < RP; ++r) {
        V t = __ldg(tw + (r - 1) * NS + k);
        if (DIR > 0) t.y = -t.y;
        w[r] = cmul(w[r], t);
      }
    }
    Dft<RP, DIR, V>::run(w);
    if (TO_REGS) {
#pragma unroll
      for (int r = 0; r < RP; ++r) v[u + r * VP] = w[r];
    } else {
      const int idxD = (vt / NS) * NS * RP + k;
#pragma unroll
      for (int r = 0; r < RP; ++r) dst[pad<V>(idxD + r * NS)] = w[r];
    }
  }
}

// Runs passes p..P-1.  `rd` is read by pass p (unless FROM_REGS), `wr` written.  Returns the
// buffer written last (so the caller's next write phase goes to the other one).
template <typename V, int NC, int R, int DIR, int p, bool FROM_REGS>
__device__ __forceinline__ V* fft_passes(V (&v)[R], V* rd, V* wr, const V* __restrict__ tw, int j, V* last) {
  constexpr int P = sched_passes(NC, R);
  constexpr int RP = sched_radix(NC, R, p), NS = sched_ns(NC, R, p);
  constexpr bool LAST = (p == P - 1);
  stockham_pass<V, NC, R, RP, NS, DIR, FROM_REGS, LAST>(v, rd, wr, tw + sched_twoff(NC, R, p), j);
  if constexpr (!LAST) {
    __syncthreads();
    return fft_passes<V, NC, R, DIR, p + 1, false>(v, wr, rd, tw, j, wr);
  } else {
    return last;
  }
}

// ------------------------------------------------------------------ block reductions
template <int NW>
__device__ __forceinline__ void block_sum2(double& a, double& b, double* red /*[2*NW]*/, int j) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((j & 31) == 0) { red[j >> 5] = a; red[NW + (j >> 5)] = b; }
  __syncthreads();
  a = 0.0; b = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) { a += red[w]; b += red[NW + w]; }
}

// ------------------------------------------------------------------ the kernel body
template <typename Real, int NC, int R>
struct Resident {
  using V = typename Cx<Real>::V;
  static constexpr int n = 2 * NC;
  static constexpr int T = NC / R;
  static constexpr int NW = T / 32;
  static constexpr int P = sched_passes(NC, R);
  static constexpr int PADN = padded_len<V>(NC);
  static_assert(T >= 32 && T % 32 == 0, "need at least one full warp");
  static_assert((NC & (NC - 1)) == 0, "power-of-two NC");

  // dynamic shared memory layout (bytes)
  static constexpr size_t off_bufA = 0;
  static constexpr size_t off_bufB = off_bufA + sizeof(V) * PADN;
  static constexpr size_t off_sin = off_bufB + sizeof(V) * PADN;
  static constexpr size_t off_isin = off_sin + sizeof(Real) * ((NC + 2) & ~1);
  static constexpr size_t off_red = off_isin + sizeof(Real) * ((NC + 2) & ~1);   // 2 slots x 2*NW doubles
  static constexpr size_t off_nbr = off_red + sizeof(double) * 4 * NW;          // NW*R V
  static constexpr size_t off_int = off_nbr + sizeof(V) * NW * R;               // NW + 8 ints
  static constexpr size_t smem_bytes = off_int + sizeof(int) * (NW + 8);

  struct Smem {
    V* bufA; V* bufB; Real* sint; Real* isin; double* red; V* nbr; int* ired;
  };

  // -------------------------------------------------------------- a2 extrema count
  // Fast path: with no zero difference, k = #{p : sign(D_p) != sign(D_p+1)} -- a plain
  // sum.  Any zero difference -> exact sequential rule (zeros dropped) in one warp.
  __device__ static int extrema(const V (&rt)[R], const Smem& sm, V*& last, int j) {
    const int lane = j & 31, w = j >> 5;
    V nb[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      nb[q].x = __shfl_down_sync(0xffffffffu, rt[q].x, 1);
      nb[q].y = __shfl_down_sync(0xffffffffu, rt[q].y, 1);
    }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < R; ++q) sm.nbr[w * R + q] = rt[q];
    }
    __syncthreads();
    if (lane == 31) {
#pragma unroll
      for (int q = 0; q < R; ++q) {
        int w2 = w + 1, q2 = q;
        if (w2 == NW) { w2 = 0; q2 = q + 1; }
        if (q2 < R) nb[q] = sm.nbr[w2 * R + q2];
      }
    }
    int cnt = 0;
    bool zero = false;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int m = j + T * q;
      const Real d0 = rt[q].y - rt[q].x;  // D_{2m}
      zero |= (d0 == (Real)0);
      if (m < NC - 1) {
        const Real d1 = nb[q].x - rt[q].y;  // D_{2m+1}
        const Real d2 = nb[q].y - nb[q].x;  // D_{2m+2} (checked for zero by pair m+1)
        zero |= (d1 == (Real)0);
        cnt += ((d0 > (Real)0) != (d1 > (Real)0)) + ((d1 > (Real)0) != (d2 > (Real)0));
      }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) sm.ired[w] = cnt;
    const int anyzero = __syncthreads_or(zero);
    int total = 0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) total += sm.ired[ww];
    if (anyzero) total = extrema_exact(rt, sm, last, j);
    return total;
  }

  // Exact rule with zero differences dropped (reading A4), one warp, ordered monoid
  // (first sign, last sign, changes) over 32 contiguous chunks.
  __device__ static int extrema_exact(const V (&rt)[R], const Smem& sm, V*& last, int j) {
    V* buf = (last == sm.bufA) ? sm.bufB : sm.bufA;
#pragma unroll
    for (int q = 0; q < R; ++q) buf[pad<V>(j + T * q)] = rt[q];
    last = buf;
    __syncthreads();
    if (j < 32) {
      constexpr int CH = NC / 32;  // pairs per lane
      int first = 0, lastsg = 0, c = 0;
      const int m0 = j * CH;
      Real prev = buf[pad<V>(m0)].x;
      for (int p = 2 * m0 + 1; p <= 2 * (m0 + CH) && p < n; ++p) {
        const V pr = buf[pad<V>(p >> 1)];
        const Real x = (p & 1) ? pr.y : pr.x;
        const Real d = x - prev;
        prev = x;
        if (d == (Real)0) continue;
        const int sg = d > (Real)0 ? 1 : -1;
        if (first == 0) first = sg;
        if (lastsg != 0 && sg != lastsg) ++c;
        lastsg = sg;
      }
      // ordered fold over lanes 0..31 (lane 0 accumulates)
      int F = __shfl_sync(0xffffffffu, first, 0), Ls = __shfl_sync(0xffffffffu, lastsg, 0),
          C = __shfl_sync(0xffffffffu, c, 0);
      for (int l = 1; l < 32; ++l) {
        const int f2 = __shfl_sync(0xffffffffu, first, l), l2 = __shfl_sync(0xffffffffu, lastsg, l),
                  c2 = __shfl_sync(0xffffffffu, c, l);
        C += c2 + ((Ls != 0 && f2 != 0 && Ls != f2) ? 1 : 0);
        if (F == 0) F = f2;
        if (l2 != 0) Ls = l2;
      }
      if (j == 0) sm.ired[NW] = C;
    }
    __syncthreads();
    return sm.ired[NW];
  }

  // -------------------------------------------------------------- a3 filter length
  __device__ static int filter_half_length(const Params& p, int k) {
    const double t = __dmul_rn(p.xi, (double)n);   // fl(xi * n), never contracted (A8)
    const double u = __ddiv_rn(t, (double)k);      // fl(fl(xi n)/k)
    long long q = (long long)floor(u);
    long long L = p.window ? 2 * q : q;
    const long long Lmax = (n - 1) / 4;
    if (L < 2) L = 2;
    if (L > Lmax) L = Lmax;
    return (int)L;
  }

  // -------------------------------------------------------------- a4 window spectrum
  // w_hat_k = [sin(pi r/n) / (L sin(pi k/n))]^4, r = min(Lk mod n, n - Lk mod n), k in [0, n/2].
  __device__ static Real what(const Smem& sm, int L, Real invL, int k) {
    if (k == 0) return (Real)1;
    const int m = (int)(((long long)L * k) & (n - 1));
    const int r = min(m, n - m);
    const Real s = sm.sint[r] * sm.isin[k] * invL;
    const Real s2 = s * s;
    return s2 * s2;
  }

  // -------------------------------------------------------------- a5 stopping search (one probe)
  // P(N) = sum c_k a_k^{2(N-1)} |X_k|^2, Q(N) = sum c_k w_k^2 a_k^{2(N-1)} |X_k|^2 (fp64 accumulation)
  // Also returns d_k = a_k^N for the thread's bins (used when N = the probe).  The thread's R+1 bins
  // are processed together (powers by squaring over the bits of the uniform exponent N-1) for ILP.
  static constexpr int NB = R + 1;  // R/2 bins k, R/2 mirrors NC-k, + the middle bin (thread 0 only)
  __device__ static void probe(const V (&Xa)[R / 2], const V (&Xb)[R / 2], const V& Xm, const Smem& sm, int L,
                               Real invL, int N, double& P, double& Q, Real (&dA)[R / 2], Real (&dB)[R / 2],
                               Real& dM, double* red, int j) {
    double a[NB], e[NB], wv[NB], pk[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      int kk;
      V X;
      if (i < R / 2) { kk = j + T * i; X = Xa[i]; }
      else if (i < R) { kk = NC - (j + T * (i - R / 2)); X = Xb[i - R / 2]; }
      else { kk = NC / 2; X = Xm; }
      const Real w = what(sm, L, invL, kk);
      const Real av = fminf_t(fmaxf_t((Real)1 - w, (Real)0), (Real)1);
      a[i] = (double)av;
      wv[i] = (double)w;
      const double c = (kk == 0 || kk == NC) ? 1.0 : 2.0;
      pk[i] = (i < R || j == 0) ? c * ((double)X.x * (double)X.x + (double)X.y * (double)X.y) : 0.0;
      e[i] = 1.0;
    }
    // e = a^(N-1) by squaring (exponent uniform across the block: no divergence)
    {
      double b[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) b[i] = a[i];
      int ex = N - 1;
      while (ex) {
        if (ex & 1) {
#pragma unroll
          for (int i = 0; i < NB; ++i) e[i] *= b[i];
        }
        ex >>= 1;
        if (ex) {
#pragma unroll
          for (int i = 0; i < NB; ++i) b[i] *= b[i];
        }
      }
    }
    P = 0.0; Q = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const double x = e[i] * e[i];
      const double px = pk[i] * x;
      P += px;
      Q += px * (wv[i] * wv[i]);
      const Real d = (Real)(e[i] * a[i]);
      if (i < R / 2) dA[i]= d; else if (i < R) dB[i - R / 2] = d; else dM = d;
    }
    block_sum2<NW>(P, Q, red, j);
  }

  __device__ static Real fminf_t(Real a, Real b) { return a < b ? a : b; }
  __device__ static Real fmaxf_t(Real a, Real b) { return a > b ? a : b; }

  __device__ static int search(const V (&Xa)[R / 2], const V (&Xb)[R / 2], const V& Xm, const Smem& sm, int L,
                               const Params& p, Real (&dA)[R / 2], Real (&dB)[R / 2], Real& dM, int& slot, int j) {
    const Real invL = (Real)1 / (Real)L;
    double Pv, Qv;
    const int cap = p.max_inner;
    probe(Xa, Xb, Xm, sm, L, invL, cap, Pv, Qv, dA, dB, dM, sm.red + slot * 2 * NW, j);
    slot ^= 1;
    if (!(Qv <= p.delta2 * Pv)) return cap;
    int lo = 0, hi = cap, lastN = cap;  // invariant: pass(hi), !pass(lo) (lo = 0 is virtual)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      probe(Xa, Xb, Xm, sm, L, invL, mid, Pv, Qv, dA, dB, dM, sm.red + slot * 2 * NW, j);
      slot ^= 1;
      lastN = mid;
      if (Qv <= p.delta2 * Pv) hi = mid; else lo = mid;
    }
    if (lastN != hi) {  // recompute d_k = a_k^hi (dA/dB hold the last probe's N)
      double Pd, Qd;
      probe(Xa, Xb, Xm, sm, L, invL, hi, Pd, Qd, dA, dB, dM, sm.red + slot * 2 * NW, j);
      slot ^= 1;
    }
    return hi;
  }

  // -------------------------------------------------------------- real-FFT pre/post processing
  // w_k = e^{+2 pi i k/n} = (sin(pi (n/2 - 2k)/n), sin(pi 2k/n)), k <= n/4
  __device__ static V wk(const Smem& sm, int k) { return V{sm.sint[NC - 2 * k], sm.sint[2 * k]}; }

  // forward: from Z (NC-point FFT of z) to X_k, X_{NC-k}
  __device__ static void post_forward(V P, V Q, V w, V& Xk, V& Xmk) {
    const Real h = (Real)0.5;
    const V E = V{h * (P.x + Q.x), h * (P.y - Q.y)};       // (P + Q*)/2
    const V D = V{h * (P.x - Q.x), h * (P.y + Q.y)};       // (P - Q*)/2
    const V O = V{D.y, -D.x};                              // D / i
    const V wO = cmul(cconj(w), O);                         // e^{-2 pi i k/n} O
    Xk = cadd(E, wO);
    Xmk = cconj(csub(E, wO));
  }
  // inverse: from A = D_k, B = D_{NC-k} (already scaled by 1/n) to Z_k, Z_{NC-k}
  __device__ static void pre_inverse(V A, V B, V w, V& Zk, V& Zmk) {
    const V S = V{A.x + B.x, A.y - B.y};    // A + B*
    const V D = V{A.x - B.x, A.y + B.y};    // A - B*
    const V Tm = mul_i<1>(cmul(w, D));      // i w (A - B*)
    Zk = cadd(S, Tm);
    Zmk = cconj(csub(S, Tm));
  }

  // forward rfft of the registers rt (pairs at m = j + T q) -> spectrum in pair layout
  __device__ static void rfft(const V (&rt)[R], V (&Xa)[R / 2], V (&Xb)[R / 2], V& Xm, const Smem& sm,
                              const V* __restrict__ tw, V*& last, int j) {
    V v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = rt[q];
    V* wr = (last == sm.bufA) ? sm.bufB : sm.bufA;
    V* rd = (wr == sm.bufA) ? sm.bufB : sm.bufA;
    V* lw = fft_passes<V, NC, R, -1, 0, true>(v, rd, wr, tw, j, wr);
    // Z -> the buffer not written last
    V* zb = (lw == sm.bufA) ? sm.bufB : sm.bufA;
#pragma unroll
    for (int q = 0; q < R; ++q) zb[pad<V>(j + T * q)] = v[q];
    last = zb;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < R / 2; ++q) {
      const int k = j + T * q;
      const V P = zb[pad<V>(k)];
      const V Q = zb[pad<V>((NC - k) & (NC - 1))];
      post_forward(P, Q, wk(sm, k), Xa[q], Xb[q]);
    }
    if (j == 0) {
      const V P = zb[pad<V>(NC / 2)];
      Xm = cconj(P);
    }
  }

  // inverse: spectrum D (pair layout, pre-scaled by 1/n) -> time-domain pairs in v (m = j + T q)
  __device__ static void irfft(const V (&Da)[R / 2], const V (&Db)[R / 2], const V& Dm, V (&v)[R], const Smem& sm,
                               const V* __restrict__ tw, V*& last, int j) {
    V* zb = (last == sm.bufA) ? sm.bufB : sm.bufA;
#pragma unroll
    for (int q = 0; q < R / 2; ++q) {
      const int k = j + T * q;
      V Zk, Zmk;
      pre_inverse(Da[q], Db[q], wk(sm, k), Zk, Zmk);
      zb[pad<V>(k)] = Zk;
      if (k != 0) zb[pad<V>(NC - k)] = Zmk;
    }
    if (j == 0) zb[pad<V>(NC / 2)] = V{(Real)2 * Dm.x, -(Real)2 * Dm.y};  // 2 conj(D_mid)
    __syncthreads();
    V* other = (zb == sm.bufA) ? sm.bufB : sm.bufA;
    last = fft_passes<V, NC, R, 1, 0, false>(v, zb, other, tw, j, zb);
  }

  // -------------------------------------------------------------- one signal, all IMFs
  __device__ static void decompose_one(const Real* __restrict__ s, Real* __restrict__ out, int32_t* count,
                                       int32_t* lens, int32_t* iters, const Params& p, const Smem& sm,
                                       const V* __restrict__ tw, int& slot, V*& last, int j) {
    V rt[R];
    bool finite = true;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      rt[q] = __ldcs(reinterpret_cast<const V*>(s) + j + T * q);
      finite &= isfinite(rt[q].x) && isfinite(rt[q].y);
    }
    const size_t slot_stride = (size_t)n;
    if (!__syncthreads_and(finite)) {
      for (int m = 0; m <= p.max_imfs; ++m)
#pragma unroll
        for (int q = 0; q < R; ++q) __stcs(reinterpret_cast<V*>(out + m * slot_stride) + j + T * q, V{0, 0});
      for (int m = j; m < p.max_imfs; m += T) { lens[m] = 0; iters[m] = 0; }
      if (j == 0) *count = -1;
      return;
    }
    V Xa[R / 2], Xb[R / 2], Xm{0, 0};
    rfft(rt, Xa, Xb, Xm, sm, tw, last, j);
    int k = extrema(rt, sm, last, j);
    int M = 0;
    const Real invn = (Real)1 / (Real)n;
    while (M < p.max_imfs && k >= 2) {
      const int L = filter_half_length(p, k);
      Real dA[R / 2], dB[R / 2], dM = 0;
      const int N = search(Xa, Xb, Xm, sm, L, p, dA, dB, dM, slot, j);
      // damping: D = d X / n (IMF spectrum), X <- (1 - d) X
      V Da[R / 2], Db[R / 2], Dmv{0, 0};
#pragma unroll
      for (int q = 0; q < R / 2; ++q) {
        const Real sa = dA[q] * invn, sb = dB[q] * invn;
        Da[q] = V{Xa[q].x * sa, Xa[q].y * sa};
        Db[q] = V{Xb[q].x * sb, Xb[q].y * sb};
        const Real ra = (Real)1 - dA[q], rb = (Real)1 - dB[q];
        Xa[q] = V{Xa[q].x * ra, Xa[q].y * ra};
        Xb[q] = V{Xb[q].x * rb, Xb[q].y * rb};
      }
      if (j == 0) {
        const Real sm_ = dM * invn, rm = (Real)1 - dM;
        Dmv = V{Xm.x * sm_, Xm.y * sm_};
        Xm = V{Xm.x * rm, Xm.y * rm};
      }
      V v[R];
      irfft(Da, Db, Dmv, v, sm, tw, last, j);
      Real* o = out + (size_t)M * slot_stride;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        __stcs(reinterpret_cast<V*>(o) + j + T * q, v[q]);
        rt[q] = csub(rt[q], v[q]);
      }
      if (j == 0) { lens[M] = 2 * L; iters[M] = N; }
      ++M;
      k = extrema(rt, sm, last, j);
    }
    // trend in slot M, zeros after (A12)
#pragma unroll
    for (int q = 0; q < R; ++q) __stcs(reinterpret_cast<V*>(out + (size_t)M * slot_stride) + j + T * q, rt[q]);
    for (int m = M + 1; m <= p.max_imfs; ++m)
#pragma unroll
      for (int q = 0; q < R; ++q) __stcs(reinterpret_cast<V*>(out + (size_t)m * slot_stride) + j + T * q, V{0, 0});
    for (int m = M + j; m < p.max_imfs; m += T) { lens[m] = 0; iters[m] = 0; }
    if (j == 0) *count = M;
  }

  __device__ static Smem carve(char* base) {
    Smem sm;
    sm.bufA = reinterpret_cast<V*>(base + off_bufA);
    sm.bufB = reinterpret_cast<V*>(base + off_bufB);
    sm.sint = reinterpret_cast<Real*>(base + off_sin);
    sm.isin = reinterpret_cast<Real*>(base + off_isin);
    sm.red = reinterpret_cast<double*>(base + off_red);
    sm.nbr = reinterpret_cast<V*>(base + off_nbr);
    sm.ired = reinterpret_cast<int*>(base + off_int);
    return sm;
  }

  __device__ static void load_tables(const Smem& sm, const Real* __restrict__ sintab, const Real* __restrict__ isintab,
                                     int j) {
    for (int i = j; i <= NC; i += T) { sm.sint[i] = sintab[i]; sm.isin[i] = isintab[i]; }
    __syncthreads();
  }
};

// ------------------------------------------------------------------ kernels
template <typename Real, int NC, int R>
__global__ void __launch_bounds__(NC / R, (NC / R) <= 256 ? FIF_MINB : 1)
fif_resident_kernel(const Real* __restrict__ sig, Real* __restrict__ imfs, int32_t* __restrict__ count,
                    int32_t* __restrict__ lens, int32_t* __restrict__ iters, const Real* __restrict__ sintab,
                    const Real* __restrict__ isintab, const typename Cx<Real>::V* __restrict__ tw, Params p) {
  using K = Resident<Real, NC, R>;
  extern __shared__ __align__(16) char smem_raw[];
  const typename K::Smem sm = K::carve(smem_raw);
  const int j = threadIdx.x;
  K::load_tables(sm, sintab, isintab, j);
  int slot = 0;
  typename Cx<Real>::V* last = sm.bufA;
  for (int64_t b = blockIdx.x; b < p.batch; b += gridDim.x) {
    K::decompose_one(sig + b * K::n, imfs + b * (int64_t)(p.max_imfs + 1) * K::n, count + b,
                     lens + b * p.max_imfs, iters + b * p.max_imfs, p, sm, tw, slot, last, j);
  }
}

// test hook kernels (same device code) --------------------------------------------------------
template <typename Real, int NC, int R>
__global__ void __launch_bounds__(NC / R) fif_test_rfft_kernel(const Real* __restrict__ in, Real* __restrict__ out,
                                                             int64_t batch, const Real* __restrict__ sintab,
                                                             const Real* __restrict__ isintab,
                                                             const typename Cx<Real>::V* __restrict__ tw) {
  using K = Resident<Real, NC, R>;
  using V = typename Cx<Real>::V;
  extern __shared__ __align__(16) char smem_raw[];
  const typename K::Smem sm = K::carve(smem_raw);
  const int j = threadIdx.x;
  K::load_tables(sm, sintab, isintab, j);
  V* last = sm.bufA;
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    V rt[R], Xa[R / 2], Xb[R / 2], Xm{0, 0};
    for (int q = 0; q < R; ++q) rt[q] = reinterpret_cast<const V*>(in + b * K::n)[j + K::T * q];
    K::rfft(rt, Xa, Xb, Xm, sm, tw, last, j);
    V* o = reinterpret_cast<V*>(out + b * (K::n + 2));
    for (int q = 0; q < R / 2; ++q) {
      const int k = j + K::T * q;
      o[k] = Xa[q];
      o[NC - k] = Xb[q];
    }
    if (j == 0) o[NC / 2] = Xm;
    __syncthreads();
  }
}

template <typename Real, int NC, int R>
__global__ void __launch_bounds__(NC / R) fif_test_irfft_kernel(const Real* __restrict__ in, Real* __restrict__ out,
                                                              int64_t batch, const Real* __restrict__ sintab,
                                                              const Real* __restrict__ isintab,
                                                              const typename Cx<Real>::V* __restrict__ tw) {
  using K = Resident<Real, NC, R>;
  using V = typename Cx<Real>::V;
  extern __shared__ __align__(16) char smem_raw[];
  const typename K::Smem sm = K::carve(smem_raw);
  const int j = threadIdx.x;
  K::load_tables(sm, sintab, isintab, j);
  V* last = sm.bufA;
  const Real invn = (Real)1 / (Real)K::n;
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    const V* x = reinterpret_cast<const V*>(in + b * (K::n + 2));
    V Da[R / 2], Db[R / 2], Dm{0, 0}, v[R];
    for (int q = 0; q < R / 2; ++q) {
      const int k = j + K::T * q;
      Da[q] = V{x[k].x * invn, x[k].y * invn};
      Db[q] = V{x[NC - k].x * invn, x[NC - k].y * invn};
    }
    if (j == 0) Dm = V{x[NC / 2].x * invn, x[NC / 2].y * invn};
    K::irfft(Da, Db, Dm, v, sm, tw, last, j);
    for (int q = 0; q < R; ++q) reinterpret_cast<V*>(out + b * K::n)[j + K::T * q] = v[q];
    __syncthreads();
  }
}

template <typename Real, int NC, int R>
__global__ void __launch_bounds__(NC / R) fif_test_extrema_kernel(const Real* __restrict__ in, int32_t* __restrict__ kout,
                                                                int64_t batch) {
  using K = Resident<Real, NC, R>;
  using V = typename Cx<Real>::V;
  extern __shared__ __align__(16) char smem_raw[];
  const typename K::Smem sm = K::carve(smem_raw);
  const int j = threadIdx.x;
  V* last = sm.bufA;
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    V rt[R];
    for (int q = 0; q < R; ++q) rt[q] = reinterpret_cast<const V*>(in + b * K::n)[j + K::T * q];
    const int k = K::extrema(rt, sm, last, j);
    if (j == 0) kout[b] = k;
    __syncthreads();
  }
}

template <typename Real, int NC, int R>
__global__ void __launch_bounds__(NC / R) fif_test_window_kernel(Real* __restrict__ out, int L,
                                                               const Real* __restrict__ sintab,
                                                               const Real* __restrict__ isintab) {
  using K = Resident<Real, NC, R>;
  extern __shared__ __align__(16) char smem_raw[];
  const typename K::Smem sm = K::carve(smem_raw);
  const int j = threadIdx.x;
  K::load_tables(sm, sintab, isintab, j);
  const Real invL = (Real)1 / (Real)L;
  for (int k = j; k <= NC; k += K::T) out[k] = K::what(sm, L, invL, k);
}

template <typename Real, int NC, int R>
__global__ void __launch_bounds__(NC / R) fif_test_inner_kernel(const Real* __restrict__ in, Real* __restrict__ out,
                                                              int32_t* __restrict__ Nout, int64_t batch, int L,
                                                              const Real* __restrict__ sintab,
                                                              const Real* __restrict__ isintab,
                                                              const typename Cx<Real>::V* __restrict__ tw, Params p) {
  using K = Resident<Real, NC, R>;
  using V = typename Cx<Real>::V;
  extern __shared__ __align__(16) char smem_raw[];
  const typename K::Smem sm = K::carve(smem_raw);
  const int j = threadIdx.x;
  K::load_tables(sm, sintab, isintab, j);
  V* last = sm.bufA;
  int slot = 0;
  const Real invn = (Real)1 / (Real)K::n;
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    V rt[R], Xa[R / 2], Xb[R / 2], Xm{0, 0};
    for (int q = 0; q < R; ++q) rt[q] = reinterpret_cast<const V*>(in + b * K::n)[j + K::T * q];
    K::rfft(rt, Xa, Xb, Xm, sm, tw, last, j);
    Real dA[R / 2], dB[R / 2], dM = 0;
    const int N = K::search(Xa, Xb, Xm, sm, L, p, dA, dB, dM, slot, j);
    V Da[R / 2], Db[R / 2], Dmv{0, 0}, v[R];
    for (int q = 0; q < R / 2; ++q) {
      Da[q] = V{Xa[q].x * dA[q] * invn, Xa[q].y * dA[q] * invn};
      Db[q] = V{Xb[q].x * dB[q] * invn, Xb[q].y * dB[q] * invn};
    }
    if (j == 0) Dmv = V{Xm.x * dM * invn, Xm.y * dM * invn};
    K::irfft(Da, Db, Dmv, v, sm, tw, last, j);
    for (int q = 0; q < R; ++q) reinterpret_cast<V*>(out + b * K::n)[j + K::T * q] = v[q];
    if (j == 0) Nout[b] = N;
    __syncthreads();
  }
}

}  // namespace fifgpu
