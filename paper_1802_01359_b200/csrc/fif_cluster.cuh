// fif_cluster.cuh -- the cluster-resident FIF kernel for sm_100a: one signal per thread-block CLUSTER of P
// CTAs (P = 2, 4, 8), for n beyond one CTA (configs 2 and 4: n/2 = P Q, Q = 4096 fp64 / 8192 fp32).
//
// As in the resident kernel (fif_resident.cuh) the remainder r and its spectrum r_hat stay ON CHIP for all
// IMFs -- spread over the cluster's registers -- so HBM sees only the compulsory traffic: s read once, every
// IMF and the trend written once.  The difference is the transform: an n/2 = P Q point complex FFT as a
// four-step FFT over the cluster ("U^T s is the DFT of s ... FFT"):
//   bins     k = c + P k1      CTA c holds the residue class c mod P, local index k1 = t + T r
//                              (thread t, register r) -- the local Q-point transform is a CTA's own;
//   time     m = q + Q p,      q = j W + u T + t (W = Q/P, U = 8/P): CTA j holds P chunks of W
//                              consecutive points (register r = u P + p), so IMF stores stay coalesced
//                              and the extrema count needs only the chunk ends from its neighbours.
// Inverse (per IMF): damping -> real-IFFT pre-processing (bin k with NC - k, which lives in CTA P - c: the
// partner's damped spectrum is published to an L2-resident scratch and brought back by ONE bulk copy) ->
// local Q-point IFFT -> twiddle e^{+2 pi i c q/NC} -> the cluster transpose: every CTA writes its
// W-slices to the destinations' scratch regions, cluster barrier, each destination lands its region
// with ONE cp.async.bulk (the TMA engine) -> P-point IDFT in registers.  The forward transform (once)
// runs the same steps backwards.  Reductions (Parseval sums, extrema partials) go through distributed
// shared memory and the cluster barrier; every CTA then takes the same decisions.
//
// Steps and readings are those of fif_resident.cuh:
//   a1 forward rfft
//   a2 extrema count           (A4)        a3 L rule (A1, A3, A8)
//   a4 window spectrum         closed form of DESIGN.md §4, sines by geometric recurrences from a
//                              two-level table of e^{i pi j/n}
//   a5 stopping search         cap probe, 4-ary fp32 hint verified in fp64, fp64 bisection fallback
//                              (Parseval :175-180; P7)
//   a6 damping + C2R IFFT + remainder update
//   a7 outer control, trend, zero fill
#pragma once
#include <cooperative_groups.h>

#include "fif_resident.cuh"
#include "fif_streamed.cuh"  // bulk-copy / mbarrier helpers (st::bulk_g2s ...)

namespace fifgpu {
namespace cl {
namespace cg = cooperative_groups;

// per-cluster global scratch (L2-resident: 2 NC complex per cluster)
struct Scratch {
  void* pub;   // [clusters][P][Q] V: each CTA's published (natural-order) spectrum for its mirror partner
  void* xch;   // [clusters][P][Q] V: transpose landing regions, one per destination CTA
};

template <typename Real, int Q, int P, int CAP>
struct Clu {
  using V = typename Cx<Real>::V;
  static constexpr int NC = P * Q;
  static constexpr int n = 2 * NC;
  static constexpr int R = kR;        // 8 values per thread
  static constexpr int T = Q / R;     // threads per CTA
  static constexpr int NW = T / 32;
  static constexpr int U = R / P;     // q-groups per thread in the time domain
  static constexpr int W = Q / P;     // time points per chunk (= U T)
  static constexpr int EB = 9;        // E(j) = e^{i pi j/n}, j < 2n: Eh[j >> EB] * El[j & (2^EB - 1)]
  static constexpr int NEL = 1 << EB;
  static constexpr int NEH = (2 * n) >> EB;
  static constexpr int NB = R + 1;
  static_assert(P == 2 || P == 4 || P == 8, "cluster of 2, 4 or 8 CTAs");
  static_assert(T % 32 == 0 && (Q & (Q - 1)) == 0, "power-of-two Q, whole warps");

  // ---- dynamic shared memory layout (bytes)
  static constexpr size_t oA = 0;                                   // FFT ping-pong buffers
  static constexpr size_t oB = oA + sizeof(V) * Q;
  static constexpr size_t oR = oB + sizeof(V) * Q;                  // bulk-copy landing buffer
  static constexpr size_t oEh = oR + sizeof(V) * Q;
  static constexpr size_t oEl = oEh + sizeof(double2) * NEH;
  static constexpr size_t oRed = oEl + sizeof(double2) * NEL;       // block reductions: 2 slots x 4 NW doubles
  static constexpr size_t oCred = oRed + sizeof(double) * 8 * NW;   // cluster partials: 2 slots x P x 8 doubles
  static constexpr size_t oBnd = oCred + sizeof(double) * 2 * P * 8;  // chunk ends: [P src][P p][4] doubles
  static constexpr size_t oNbr = oBnd + sizeof(double) * P * P * 4;   // warp lane-0 values [NW][R]
  static constexpr size_t oInt = oNbr + sizeof(Real) * NW * R;        // ints: [NW] counts, [NW] masks, misc
  static constexpr size_t oBar = (oInt + sizeof(int) * (2 * NW + 2 * P + 8) + 15) & ~(size_t)15;
  static constexpr size_t smem_bytes = oBar + 32;  // bar (bulk landings), cbar[2] (cluster reductions)

  struct Sm {
    V *A, *B, *Rl;
    double2 *Eh, *El;
    double* red;
    double* cred;
    double* bnd;
    Real* nbr;
    int* ints;
    uint64_t* bar;
    uint64_t* cbar;  // [2] reduction slots: each CTA's partials land by st.async, counted in transaction bytes
  };
  __device__ static Sm carve(char* base) {
    Sm s;
    s.A = reinterpret_cast<V*>(base + oA);
    s.B = reinterpret_cast<V*>(base + oB);
    s.Rl = reinterpret_cast<V*>(base + oR);
    s.Eh = reinterpret_cast<double2*>(base + oEh);
    s.El = reinterpret_cast<double2*>(base + oEl);
    s.red = reinterpret_cast<double*>(base + oRed);
    s.cred = reinterpret_cast<double*>(base + oCred);
    s.bnd = reinterpret_cast<double*>(base + oBnd);
    s.nbr = reinterpret_cast<Real*>(base + oNbr);
    s.ints = reinterpret_cast<int*>(base + oInt);
    s.bar = reinterpret_cast<uint64_t*>(base + oBar);
    s.cbar = s.bar + 1;
    return s;
  }

  // ---- tables: e^{i pi j/n}, 0 <= j < 2n (exact integer index arithmetic, one complex product)
  __device__ static double2 E(const Sm& s, unsigned j) {
    j &= (unsigned)(2 * n - 1);
    return cmul(s.Eh[j >> EB], s.El[j & (NEL - 1)]);
  }

  // ---- cluster-wide sum of M doubles (deterministic: block totals, then the P partials in rank order).
  // No cluster barrier: every CTA stores its partials into every CTA's slot with st.async, whose bytes
  // complete a transaction count on the destination's mbarrier (the local arrival announces how many);
  // each CTA waits on its own barrier only.  `slot` carries the alternating slot (bit 0) and the phase
  // parity of each slot's barrier (bits 1, 2); a slot is reused two reductions later, when every CTA has
  // necessarily consumed it.  `extra`: bytes other st.async writes (chunk ends) add to this reduction.
  __device__ static uint32_t mapa(uint32_t a, int r) {
    uint32_t x;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(x) : "r"(a), "r"(r));
    return x;
  }
  __device__ static void st_async(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n"
                 ::"r"(raddr), "l"(__double_as_longlong(v)), "r"(rbar) : "memory");
  }
  template <int M, typename S>
  __device__ static void csum_t(S (&v)[M], const Sm& s, int& slot, int rank, int t, uint32_t extra) {
    static_assert(M <= 8, "");
    const int sl = slot & 1;
    const uint32_t ph = ((uint32_t)slot >> (1 + sl)) & 1u;
    slot ^= 1 | (2 << sl);
    S* red = reinterpret_cast<S*>(s.red + sl * 4 * NW);
    double* cr = s.cred + sl * P * 8;
    block_sum<NW, M>(v, red, t);
    if (t == 0) st::mbar_expect_tx(&s.cbar[sl], (uint32_t)(P * M * 8) + extra);
    if (t < P) {
      const uint32_t ra = mapa(st::smem_u32(cr + rank * 8), t), rb = mapa(st::smem_u32(&s.cbar[sl]), t);
#pragma unroll
      for (int i = 0; i < M; ++i) st_async(ra + 8 * i, (double)v[i], rb);
    }
    st::mbar_wait(&s.cbar[sl], ph);
#pragma unroll
    for (int i = 0; i < M; ++i) {
      double a = 0.0;
#pragma unroll
      for (int r = 0; r < P; ++r) a += cr[r * 8 + i];
      v[i] = (S)a;
    }
  }
  template <int M>
  __device__ static void csum(double (&v)[M], const Sm& s, cg::cluster_group&, int& slot, int rank, int t,
                              uint32_t extra = 0) {
    csum_t<M, double>(v, s, slot, rank, t, extra);
  }
  template <int M>
  __device__ static void csumf(float (&v)[M], const Sm& s, cg::cluster_group&, int& slot, int rank, int t) {
    csum_t<M, float>(v, s, slot, rank, t, 0);
  }

  // ---- bulk copy of Q contiguous complex values (L2 scratch) into the landing buffer; all threads wait
  __device__ static void land(const Sm& s, const V* src, uint32_t& phase, int t) {
    if (t == 0) {
      // the scratch was written by the cluster's threads through the generic proxy (ordered before this
      // point by the cluster barrier's release / acquire) and the landing buffer was last read by them:
      // both orderings extend to the bulk copy's async proxy through this fence
      asm volatile("fence.proxy.async;\n" ::: "memory");
      st::mbar_expect_tx(s.bar, (uint32_t)(sizeof(V) * Q));
      constexpr uint32_t kChunk = 32768;  // bytes per bulk copy (<= the instruction's size field)
      constexpr uint32_t total = (uint32_t)(sizeof(V) * Q);
      for (uint32_t off = 0; off < total; off += kChunk)
        st::bulk_g2s(reinterpret_cast<char*>(s.Rl) + off, reinterpret_cast<const char*>(src) + off,
                     total - off < kChunk ? total - off : kChunk, s.bar);
    }
    st::mbar_wait(s.bar, phase);
    phase ^= 1u;
  }

  // ---- a3 (A1, A3, A8): fl(fl(xi n)/k) in IEEE fp64, clamp [2, (n-1)/4]
  __device__ static int filter_half_length(const Params& p, int k) {
    const double tt = __dmul_rn(p.xi, (double)n);
    const double uu = __ddiv_rn(tt, (double)k);
    long long q = (long long)floor(uu);
    long long L = p.window ? 2 * q : q;
    const long long Lmax = (n - 1) / 4;
    if (L < 2) L = 2;
    if (L > Lmax) L = Lmax;
    return (int)L;
  }

  // ---- a4: w_hat for the thread's 8 bins k = c + P (t + T r) (+ the Nyquist bin on rank 0, thread 0)
  __device__ static void window(const Sm& s, int L, int c, int t, double (&w)[NB]) {
    const unsigned k0 = (unsigned)(c + P * t);
    double2 Ek = E(s, k0), Sk = E(s, (unsigned)((unsigned long long)L * k0 % (2ull * n)));
    const double2 Es = E(s, (unsigned)(P * T)), Ss = E(s, (unsigned)((unsigned long long)L * (P * T) % (2ull * n)));
    const double Ld = (double)L;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r > 0) {
        Ek = cmul(Ek, Es);
        Sk = cmul(Sk, Ss);
      }
      const double sk = fabs(Sk.y) / (Ld * Ek.y);  // sin(pi r_k/n) / (L sin(pi k/n)), k >= 1
      const double s2 = sk * sk;
      w[r] = s2 * s2;
    }
    if (c == 0 && t == 0) w[0] = 1.0;  // bin 0: rows sum to 1
    w[R] = (L & 1) ? 1.0 / (Ld * Ld * Ld * Ld) : 0.0;  // Nyquist bin NC: [sin(pi L/2) / L]^4
  }

  __device__ static double bin_p1(const V (&X)[R], const V& Xn, int c, int t, int q) {
    if (q == R) return (c == 0 && t == 0) ? 0.5 * __dmul_rn((double)Xn.x, (double)Xn.x) : 0.0;
    const double pp = __fma_rn((double)X[q].x, (double)X[q].x, __dmul_rn((double)X[q].y, (double)X[q].y));
    return (q == 0 && c == 0 && t == 0) ? 0.5 * pp : pp;
  }
  __device__ static void accum_bin(double p1, double w, double e, double& Pp, double& Qq, double& d) {
    const double px = __dmul_rn(p1, __dmul_rn(e, e));
    Pp = __dadd_rn(Pp, px);
    Qq = __fma_rn(px, __dmul_rn(w, w), Qq);
    d = __dmul_rn(e, __dsub_rn(1.0, w));
  }
  // the thread's share of (P, Q) at N and d = a^N (ECT >= 0: N - 1 at compile time)
  template <int ECT = -1>
  __device__ static void probe_part(const V (&X)[R], const V& Xn, const double (&wall)[NB], int N, int c, int t,
                                    double (&v)[2], double (&d)[NB]) {
    v[0] = 0.0;
    v[1] = 0.0;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      double a[4], e[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = 1.0 - wall[4 * g + i];
      if constexpr (ECT >= 0) upow_ct<ECT>(e, a); else upow<4>(e, a, N - 1);
#pragma unroll
      for (int i = 0; i < 4; ++i) accum_bin(bin_p1(X, Xn, c, t, 4 * g + i), wall[4 * g + i], e[i], v[0], v[1], d[4 * g + i]);
    }
    d[R] = 0.0;
    if (c == 0 && t == 0) {
      double a[1] = {1.0 - wall[R]}, e[1];
      if constexpr (ECT >= 0) upow_ct<ECT>(e, a); else upow<1>(e, a, N - 1);
      accum_bin(bin_p1(X, Xn, c, t, R), wall[R], e[0], v[0], v[1], d[R]);
    }
    v[0] *= 2.0;
    v[1] *= 2.0;
  }
  __device__ static void verify(const V (&X)[R], const V& Xn, const double (&wall)[NB], int N, double delta2, int c,
                                int t, bool& plo, bool& phi, double (&d)[NB], const Sm& s, cg::cluster_group& cl,
                                int& slot, int rank) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    const int ex = N > 1 ? N - 2 : 0;
    auto vb = [&](double p1, double w, double a, double e, double& dd) {
      const double w2 = __dmul_rn(w, w);
      const double e1 = N > 1 ? __dmul_rn(e, a) : e;
      const double x0 = __dmul_rn(p1, __dmul_rn(e, e)), x1 = __dmul_rn(p1, __dmul_rn(e1, e1));
      v[0] = __dadd_rn(v[0], x0);
      v[1] = __fma_rn(x0, w2, v[1]);
      v[2] = __dadd_rn(v[2], x1);
      v[3] = __fma_rn(x1, w2, v[3]);
      dd = __dmul_rn(e1, a);
    };
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      double a[4], e[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = 1.0 - wall[4 * g + i];
      upow<4>(e, a, ex);
#pragma unroll
      for (int i = 0; i < 4; ++i) vb(bin_p1(X, Xn, c, t, 4 * g + i), wall[4 * g + i], a[i], e[i], d[4 * g + i]);
    }
    d[R] = 0.0;
    if (c == 0 && t == 0) {
      double a[1] = {1.0 - wall[R]}, e[1];
      upow<1>(e, a, ex);
      vb(bin_p1(X, Xn, c, t, R), wall[R], a[0], e[0], d[R]);
    }
    csum<4>(v, s, cl, slot, rank, t);
    plo = (N > 1) && (v[1] <= delta2 * v[0]);
    phi = v[3] <= delta2 * v[2];
  }
  __device__ static float lg2f(float x) { float y; asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
  __device__ static float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
  // 4-ary fp32 hint (as fif_resident.cuh hint_fp32), cluster reductions
  __device__ static int hint(const V (&X)[R], const V& Xn, const double (&wall)[NB], int hi, float delta2, int c,
                             int t, const Sm& s, cg::cluster_group& cl, int& slot, int rank) {
    float l2[NB], pk[NB], pw[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const double w = wall[q], p64 = bin_p1(X, Xn, c, t, q);
      l2[q] = fmaxf(2.0f * lg2f(fmaxf((float)(1.0 - w), 0.0f)), -1e30f);
      pk[q] = (float)p64;
      pw[q] = (float)(p64 * w * w);
    }
    int lo = 0;
    while (hi - lo > 1) {
      const int D = (hi - lo + 3) >> 2;
      const float t1 = (float)(lo + D - 1), tD = (float)D;
      float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        if (i == R && !(c == 0 && t == 0)) break;
        const float x1 = ex2f(t1 * l2[i]), sx = ex2f(tD * l2[i]);
        const float x2 = x1 * sx, x3 = x2 * sx;
        v[0] += pk[i] * x1; v[1] += pw[i] * x1;
        v[2] += pk[i] * x2; v[3] += pw[i] * x2;
        v[4] += pk[i] * x3; v[5] += pw[i] * x3;
      }
      csumf<6>(v, s, cl, slot, rank, t);
      int nlo = lo, nhi = hi;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int m = lo + (i + 1) * D;
        if (m >= hi) break;
        if (v[2 * i + 1] <= delta2 * v[2 * i]) { nhi = m; break; }
        nlo = m;
      }
      lo = nlo;
      hi = nhi;
    }
    return hi;
  }

  // ---- a5: N and d = a^N for the thread's bins (every CTA of the cluster gets the same N)
  __device__ static int search(const V (&X)[R], const V& Xn, const Sm& s, int L, const Params& p, int c, int t,
                               double (&dd)[NB], cg::cluster_group& cl, int& slot, int rank) {
    double wall[NB];
    window(s, L, c, t, wall);
    const int cap = p.max_inner;
    int N = cap;
    if (p.stop == 1) {
      // N0 rule: ||U^T r||_inf = max_k |X_k| / sqrt(n) (A16), k = 0 zero eigenvalues (A17)
      double mx = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) mx = fmax(mx, (double)X[q].x * (double)X[q].x + (double)X[q].y * (double)X[q].y);
      if (c == 0 && t == 0) mx = fmax(mx, (double)Xn.x * (double)Xn.x);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      double* red = s.red + (slot & 1) * 4 * NW;
      double* cr = s.cred + (slot & 1) * P * 8;
      slot ^= 1;  // (a barrier-synchronised use: the slot's mbarrier phase is untouched)
      if ((t & 31) == 0) red[t >> 5] = mx;
      __syncthreads();
      mx = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) mx = fmax(mx, red[w]);
      if (t < P) cl.map_shared_rank(cr, t)[rank * 8] = mx;
      cl.sync();
      mx = 0.0;
#pragma unroll
      for (int r = 0; r < P; ++r) mx = fmax(mx, cr[r * 8]);
      const double rhs = p.delta / (sqrt(mx / (double)n) * sqrt((double)(n - 1)));
      N = n0_capped(rhs, cap);
      bool lo, hi;
      verify(X, Xn, wall, N, p.delta2, c, t, lo, hi, dd, s, cl, slot, rank);
    } else {
      double v[2];
      if constexpr (CAP > 0) probe_part<CAP - 1>(X, Xn, wall, cap, c, t, v, dd);
      else probe_part(X, Xn, wall, cap, c, t, v, dd);
      csum<2>(v, s, cl, slot, rank, t);
      if (v[1] <= p.delta2 * v[0]) {  // SD(cap) <= delta: the minimal passing N lies below the cap
        const int Nh = hint(X, Xn, wall, cap, (float)p.delta2, c, t, s, cl, slot, rank);
        bool plo, phi;
        verify(X, Xn, wall, Nh, p.delta2, c, t, plo, phi, dd, s, cl, slot, rank);
        if (phi && !plo) {
          N = Nh;
        } else {
          int lo = phi ? 0 : Nh, hi = phi ? Nh - 1 : cap;
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            probe_part(X, Xn, wall, mid, c, t, v, dd);
            csum<2>(v, s, cl, slot, rank, t);
            if (v[1] <= p.delta2 * v[0]) hi = mid; else lo = mid;
          }
          probe_part(X, Xn, wall, hi, c, t, v, dd);  // d = a^N (no reduction needed)
          N = hi;
        }
      }
    }
    if (p.gamma > 0.0) {  // gamma-threshold (A19)
#pragma unroll
      for (int q = 0; q < NB; ++q)
        if (dd[q] >= 1.0 - p.gamma) dd[q] = 1.0;
    }
    return N;
  }

  // ---- a2: interior extrema of r over the whole cluster (A4).  Differences inside a chunk are counted by
  // their owners (warp shuffles, warp-boundary values through shared memory); the chunk ends (t = T - 1,
  // u = U - 1: the next point lives in the next CTA, or in CTA 0's next chunk) are published with the
  // partial counts and every CTA evaluates all of them in the same order.  Any zero (or subnormal)
  // difference: the exact plateau rule on the whole remainder, staged through the scratch row `zrow`.
  __device__ static unsigned sgn_bit(double d) { return (unsigned)__double2hiint(d) >> 31; }
  __device__ static unsigned sgn_bit(float d) { return (unsigned)__float_as_int(d) >> 31; }
  __device__ static unsigned expo(double d) { return (unsigned)__double2hiint(d) & 0x7ff00000u; }
  __device__ static unsigned expo(float d) { return (unsigned)__float_as_int(d) & 0x7f800000u; }
  __device__ static int extrema(const V (&rt)[R], const Sm& s, cg::cluster_group& cl, int& slot, int rank, int t,
                                Real* zrow) {
    const int lane = t & 31, w = t >> 5;
    unsigned S0 = 0, S1 = 0, emin = 0xffffffffu;
    Real xn[R];
#pragma unroll
    for (int q = 0; q < R; ++q) xn[q] = __shfl_down_sync(0xffffffffu, rt[q].x, 1);
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const Real d0 = rt[q].y - rt[q].x;
      S0 |= sgn_bit(d0) << q;
      emin = min(emin, expo(d0));
    }
    unsigned S2 = __shfl_down_sync(0xffffffffu, S0, 1);
    int* cnts = s.ints;          // [NW]
    int* masks = s.ints + NW;    // [NW]
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < R; ++q) s.nbr[w * R + q] = rt[q].x;
      masks[w] = (int)S0;
    }
    __syncthreads();
    // successor of register q = u P + p at t = T - 1 is (t = 0, u + 1, p) in this CTA; at u = U - 1 it is in
    // another CTA (a chunk end, handled after the cluster barrier)
    unsigned valid = 0xffu;
    if (lane == 31) {
      if (w + 1 < NW) {
#pragma unroll
        for (int q = 0; q < R; ++q) xn[q] = s.nbr[(w + 1) * R + q];
        S2 = (unsigned)masks[w + 1];
      } else {
        S2 = 0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int u = q / P, pp = q % P;
          if (u + 1 < U) {
            xn[q] = s.nbr[(u + 1) * P + pp];
            S2 |= (((unsigned)masks[0] >> ((u + 1) * P + pp)) & 1u) << q;
          } else {
            valid &= ~(1u << q);  // chunk end
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const Real d1 = xn[q] - rt[q].y;
      S1 |= sgn_bit(d1) << q;
      if ((valid >> q) & 1u) emin = min(emin, expo(d1));
    }
    int cnt = __popc((S0 ^ S1) & valid) + __popc((S1 ^ S2) & valid);
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    const unsigned anyz = __any_sync(0xffffffffu, emin == 0u) ? 1u : 0u;
    if (lane == 0) cnts[w] = (int)(cnt | (anyz << 30));
    // chunk ends of this CTA: first point (t = 0, u = 0) and last point (t = T - 1, u = U - 1) of each p
    double* bmine = s.bnd + rank * P * 4;
    __syncthreads();
    int ctot = 0, z = 0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) {
      ctot += cnts[ww] & 0x3fffffff;
      z |= cnts[ww] >> 30;
    }
    if (t == 0 || t == T - 1) {
      // publish to every CTA: [src rank][p][first x, first S0 bit | last y, last S0 bit], by st.async on the
      // mbarrier of the reduction slot the partial counts use next (its byte count includes these)
      const uint32_t cb = st::smem_u32(&s.cbar[slot & 1]);
#pragma unroll
      for (int r = 0; r < P; ++r) {
        const uint32_t ra = mapa(st::smem_u32(bmine), r), rb = mapa(cb, r);
#pragma unroll
        for (int pp = 0; pp < P; ++pp) {
          const int q0 = pp, q1 = (U - 1) * P + pp;
          if (t == 0) {
            st_async(ra + (pp * 4 + 0) * 8, (double)rt[q0].x, rb);
            st_async(ra + (pp * 4 + 1) * 8, (double)((S0 >> q0) & 1u), rb);
          } else {
            st_async(ra + (pp * 4 + 2) * 8, (double)rt[q1].y, rb);
            st_async(ra + (pp * 4 + 3) * 8, (double)((S0 >> q1) & 1u), rb);
          }
        }
      }
    }
    // partial count and zero flag (rank order), then the chunk-end terms, evaluated by every CTA alike
    double pv[2] = {t == 0 ? (double)ctot : 0.0, t == 0 ? (double)z : 0.0};  // (one contribution per CTA)
    csum<2>(pv, s, cl, slot, rank, t, (uint32_t)(P * P * 4 * 8));  // (its barrier also lands the chunk ends)
    // the P x P chunk-end terms, spread over the lanes of every warp (each warp gets the same total)
    int bt = 0;
    bool bz = false;
    for (int e = lane; e < P * P; e += 32) {
      // chunk (src, pp) ends at pair m = pp Q + (src + 1) W - 1; its successor starts chunk (src + 1, pp)
      // or, for the last CTA, chunk (0, pp + 1); the signal's last pair has none
      const int src = e / P, pp = e % P;
      if (src == P - 1 && pp == P - 1) continue;
      const double* a = s.bnd + (src * P + pp) * 4;
      const double* b = src + 1 < P ? s.bnd + ((src + 1) * P + pp) * 4 : s.bnd + (0 * P + pp + 1) * 4;
      const Real d1 = (Real)b[0] - (Real)a[2];
      const unsigned s0 = a[3] != 0.0, s1 = sgn_bit(d1), s2 = b[1] != 0.0;
      bt += (int)(s0 != s1) + (int)(s1 != s2);
      bz |= expo(d1) == 0u;
    }
    const int total = (int)pv[0] + __reduce_add_sync(0xffffffffu, bt);
    const bool zero = pv[1] != 0.0 || __any_sync(0xffffffffu, bz);
    if (zero) return extrema_exact(rt, s, cl, slot, rank, t, zrow);
    return total;
  }
  // exact rule (zero differences dropped) on the whole remainder: every CTA stages its chunks into zrow
  // (the signal's trend slot, free until the trend is written), one warp of rank 0 folds it in time order
  __device__ static int extrema_exact(const V (&rt)[R], const Sm& s, cg::cluster_group& cl, int& slot, int rank,
                                      int t, Real* zrow) {
    const int j = rank;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int u = q / P, pp = q % P;
      const int m = pp * Q + j * W + u * T + t;
      reinterpret_cast<V*>(zrow)[m] = rt[q];
    }
    cl.sync();  // (release / acquire at cluster scope: the scratch writes are visible to every CTA)
    double v[1] = {0.0};
    if (rank == 0 && t < 32) {
      constexpr int CH = n / 32;  // samples per lane
      int first = 0, lastsg = 0, cc = 0;
      const int s0 = t * CH;
      Real prev = __ldcg(zrow + s0);
      for (int i = s0 + 1; i < s0 + CH + 1 && i < n; ++i) {
        const Real x = __ldcg(zrow + i);
        const Real d = x - prev;
        prev = x;
        if (d == (Real)0) continue;
        const int sg = d > (Real)0 ? 1 : -1;
        if (first == 0) first = sg;
        if (lastsg != 0 && sg != lastsg) ++cc;
        lastsg = sg;
      }
      int F = __shfl_sync(0xffffffffu, first, 0), Ls = __shfl_sync(0xffffffffu, lastsg, 0),
          C = __shfl_sync(0xffffffffu, cc, 0);
      for (int l = 1; l < 32; ++l) {
        const int f2 = __shfl_sync(0xffffffffu, first, l), l2 = __shfl_sync(0xffffffffu, lastsg, l),
                  c2 = __shfl_sync(0xffffffffu, cc, l);
        C += c2 + ((Ls != 0 && f2 != 0 && Ls != f2) ? 1 : 0);
        if (F == 0) F = f2;
        if (l2 != 0) Ls = l2;
      }
      if (t == 0) v[0] = (double)C;
    }
    csum<1>(v, s, cl, slot, rank, t);  // the count lives in rank 0's thread 0 only: the sum distributes it
    return (int)v[0];
  }

  // ---- P-point DFT over the registers of one q-group (DIR -1 forward, +1 inverse)
  template <int DIR>
  __device__ static void dftP(V* x) {
    Dft<P, DIR, V>::run(x);
  }

  // ---- forward transform of the remainder rt (time chunks) -> spectrum X (natural local bins) + Xn
  __device__ static void forward(const V (&rt)[R], V (&X)[R], V& Xn, const Sm& s, cg::cluster_group& cl,
                                 const V* __restrict__ tw, V* pub_all, V* xch_all, uint32_t& phase, int rank, int t) {
    const int j = rank;
    V v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = rt[q];
    // P-point DFTs over p (each q-group u) and the twiddle e^{-2 pi i k2 q/NC}; publish Y[k2][q] to
    // destination k2's landing region at position q (natural order for its local FFT)
#pragma unroll
    for (int u = 0; u < U; ++u) {
      dftP<-1>(v + u * P);
      const int q = j * W + u * T + t;
      const double2 e1 = E(s, (unsigned)(4 * q));  // e^{2 pi i q/NC}; the k2-th twiddle is its k2-th power
      double2 ek = e1;
#pragma unroll
      for (int k2 = 0; k2 < P; ++k2) {
        V y = v[u * P + k2];
        if (k2) {
          y = cmul(y, V{(Real)ek.x, -(Real)ek.y});
          ek = cmul(ek, e1);
        }
        xch_all[(size_t)k2 * Q + q] = y;
      }
    }
    cl.sync();  // (release / acquire at cluster scope: the scratch writes are visible to every CTA)
    land(s, xch_all + (size_t)rank * Q, phase, t);
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = s.Rl[t + T * q];
    // local Q-point DFT (natural order in and out)
    fft_passes<V, Q, -1, 0, true>(v, s.A, s.B, tw, t, s.A);
    // Hermitian post-processing with the mirror bin NC - k (partner CTA P - c) -- published, landed
    const int c = rank;
#pragma unroll
    for (int q = 0; q < R; ++q) pub_all[(size_t)c * Q + t + T * q] = v[q];
    cl.sync();  // (release / acquire at cluster scope: the scratch writes are visible to every CTA)
    const int partner = (P - c) % P;
    land(s, pub_all + (size_t)partner * Q, phase, t);
    const Real h = (Real)0.5;
    double2 e = E(s, (unsigned)(2 * (c + P * t)));        // e^{2 pi i k/n}, k = c + P (t + T q) ...
    const double2 es = E(s, (unsigned)(2 * P * T));       // ... advanced by e^{2 pi i P T/n} per register
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int k1 = t + T * q;
      const int mk1 = c == 0 ? ((Q - k1) & (Q - 1)) : (Q - 1 - k1);
      const V Pz = v[q];
      const V Qz = s.Rl[mk1];
      const V Ev = V{h * (Pz.x + Qz.x), h * (Pz.y - Qz.y)};
      const V Dv = V{h * (Pz.x - Qz.x), h * (Pz.y + Qz.y)};
      const V O = V{Dv.y, -Dv.x};
      const V wf = V{(Real)e.x, -(Real)e.y};
      X[q] = cadd(Ev, cmul(wf, O));
      e = cmul(e, es);
    }
    Xn = V{0, 0};
    if (c == 0 && t == 0) {
      const V Z0 = v[0];
      Xn = V{Z0.x - Z0.y, (Real)0};
      X[0] = V{Z0.x + Z0.y, (Real)0};
    }
  }

  // ---- inverse: damped spectrum D (pre-scaled by 1/n; Dn on rank 0 thread 0) -> time chunks in v
  __device__ static void inverse(V (&v)[R], const V& Dn, const Sm& s, cg::cluster_group& cl,
                                 const V* __restrict__ tw, V* pub_all, V* xch_all, uint32_t& phase, int rank, int t) {
    const int c = rank;
#pragma unroll
    for (int q = 0; q < R; ++q) pub_all[(size_t)c * Q + t + T * q] = v[q];
    cl.sync();  // (release / acquire at cluster scope: the scratch writes are visible to every CTA)
    const int partner = (P - c) % P;
    land(s, pub_all + (size_t)partner * Q, phase, t);
    // pre-processing: Z_k = S + i w (A - conj B), S = A + conj B, A = D_k, B = D_{NC-k}, w = e^{2 pi i k/n}
    double2 e = E(s, (unsigned)(2 * (c + P * t)));  // e^{2 pi i k/n} by recurrence over the registers
    const double2 es = E(s, (unsigned)(2 * P * T));
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int k1 = t + T * q;
      const int mk1 = c == 0 ? ((Q - k1) & (Q - 1)) : (Q - 1 - k1);
      const V A = v[q];
      const V Bv = (c == 0 && k1 == 0) ? Dn : s.Rl[mk1];
      const V S = V{A.x + Bv.x, A.y - Bv.y};
      const V Dd = V{A.x - Bv.x, A.y + Bv.y};
      const V Tm = mul_i<1>(cmul(V{(Real)e.x, (Real)e.y}, Dd));
      v[q] = cadd(S, Tm);
      e = cmul(e, es);
    }
    // local Q-point IDFT (natural order in and out) and the twiddle e^{+2 pi i c q/NC}
    fft_passes<V, Q, 1, 0, true>(v, s.A, s.B, tw, t, s.A);
    const int dstride = W;  // destination j = q / W gets its slice [c][q - j W]
    double2 wq = E(s, (unsigned)(4 * c * t));   // e^{2 pi i c q/NC}, q = t + T r
    const double2 wstep = E(s, (unsigned)(4 * c * T));
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = t + T * r;
      V y = v[r];
      if (c) {
        y = cmul(y, V{(Real)wq.x, (Real)wq.y});
        wq = cmul(wq, wstep);
      }
      const int jd = q / dstride;
      xch_all[(size_t)jd * Q + (size_t)c * W + (q - jd * W)] = y;
    }
    cl.sync();  // (release / acquire at cluster scope: the scratch writes are visible to every CTA)
    land(s, xch_all + (size_t)rank * Q, phase, t);
    // P-point IDFTs over k2 for each of the thread's q-groups -> z[q + Q p]
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int k2 = 0; k2 < P; ++k2) v[u * P + k2] = s.Rl[k2 * W + u * T + t];
      dftP<1>(v + u * P);
    }
  }

  // ---- one signal, all IMFs (every CTA of the cluster runs this with its own rank)
  __device__ static void decompose_one(const Real* __restrict__ sig, Real* __restrict__ out, int32_t* count,
                                       int32_t* lens, int32_t* iters, const Params& p, const Sm& s,
                                       cg::cluster_group& cl, const V* __restrict__ tw, V* pub_all, V* xch_all,
                                       uint32_t& phase, int& slot, int rank, int t) {
    const int j = rank;
    const size_t slot_stride = (size_t)n;
    V rt[R];
    bool finite = true;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int u = q / P, pp = q % P;
      const int m = pp * Q + j * W + u * T + t;
      rt[q] = __ldcs(reinterpret_cast<const V*>(sig) + m);
      finite &= isfinite(rt[q].x) && isfinite(rt[q].y);
    }
    double fv[1] = {finite ? 0.0 : 1.0};
    csum<1>(fv, s, cl, slot, rank, t);
    auto store = [&](int mslot, const V (&x)[R]) {
      V* o = reinterpret_cast<V*>(out + (size_t)mslot * slot_stride);
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int u = q / P, pp = q % P;
        __stcs(o + pp * Q + j * W + u * T + t, x[q]);
      }
    };
    if (fv[0] != 0.0) {
      V zz[R];
#pragma unroll
      for (int q = 0; q < R; ++q) zz[q] = V{0, 0};
      for (int m = 0; m <= p.max_imfs; ++m) store(m, zz);
      if (rank == 0) {
        for (int m = t; m < p.max_imfs; m += T) { lens[m] = 0; iters[m] = 0; }
        if (t == 0) *count = -1;
      }
      return;
    }
    Real* zrow = out + (size_t)p.max_imfs * slot_stride;  // trend slot: scratch of the exact extrema rule
    V X[R], Xn{0, 0};
    forward(rt, X, Xn, s, cl, tw, pub_all, xch_all, phase, rank, t);
    int k = extrema(rt, s, cl, slot, rank, t, zrow);
    int M = 0;
    const Real invn = (Real)1 / (Real)n;
    while (M < p.max_imfs && k >= 2) {
      const int L = filter_half_length(p, k);
      // the remainder is idle through the search and the inverse transform: it waits in the IMF slot it is
      // about to be replaced by (L2-resident, the same lines are overwritten by the IMF), which keeps the
      // search's and the FFT's register peaks free of it
      {
        V* o = reinterpret_cast<V*>(out + (size_t)M * slot_stride);
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int u = q / P, pp = q % P;
          __stcg(o + pp * Q + j * W + u * T + t, rt[q]);
        }
      }
      double dd[NB];
      const int N = search(X, Xn, s, L, p, rank, t, dd, cl, slot, rank);
      V v[R], Dn{0, 0};
#pragma unroll
      for (int q = 0; q < R; ++q) {
        v[q] = cscale(X[q], (Real)dd[q] * invn);
        X[q] = cscale(X[q], (Real)1 - (Real)dd[q]);
      }
      if (rank == 0 && t == 0) {
        Dn = cscale(Xn, (Real)dd[R] * invn);
        Xn = cscale(Xn, (Real)1 - (Real)dd[R]);
      }
      inverse(v, Dn, s, cl, tw, pub_all, xch_all, phase, rank, t);
      {
        const V* o = reinterpret_cast<const V*>(out + (size_t)M * slot_stride);
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int u = q / P, pp = q % P;
          rt[q] = csub(__ldcg(o + pp * Q + j * W + u * T + t), v[q]);
        }
      }
      store(M, v);
      if (rank == 0 && t == 0) { lens[M] = 2 * L; iters[M] = N; }
      ++M;
      if (M < p.max_imfs) k = extrema(rt, s, cl, slot, rank, t, zrow);
    }
    store(M, rt);  // trend (A12)
    V zz[R];
#pragma unroll
    for (int q = 0; q < R; ++q) zz[q] = V{0, 0};
    for (int m = M + 1; m <= p.max_imfs; ++m) store(m, zz);
    if (rank == 0) {
      for (int m = M + t; m < p.max_imfs; m += T) { lens[m] = 0; iters[m] = 0; }
      if (t == 0) *count = M;
    }
  }
};

// ------------------------------------------------------------------ kernel
// grid = clusters x P CTAs (cluster dims set at launch); cluster g decomposes signals g, g + G, ...
template <typename Real, int Q, int P, int CAP>
__global__ void __launch_bounds__(Q / kR, 1)
fif_cluster_kernel(const Real* __restrict__ sig, Real* __restrict__ imfs, int32_t* __restrict__ count,
                   int32_t* __restrict__ lens, int32_t* __restrict__ iters, const double2* __restrict__ Eh,
                   const double2* __restrict__ El, const typename Cx<Real>::V* __restrict__ tw, Scratch scr,
                   Params p) {
  using K = Clu<Real, Q, P, CAP>;
  using V = typename Cx<Real>::V;
  extern __shared__ __align__(16) char smem_raw[];
  const typename K::Sm s = K::carve(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int t = threadIdx.x;
  const int64_t G = gridDim.x / P, gid = blockIdx.x / P;
  for (int i = t; i < K::NEH; i += K::T) s.Eh[i] = Eh[i];
  for (int i = t; i < K::NEL; i += K::T) s.El[i] = El[i];
  if (t == 0) {
    st::mbar_init(s.bar, 1);
    st::mbar_init(&s.cbar[0], 1);
    st::mbar_init(&s.cbar[1], 1);
    st::mbar_fence_init();
  }
  __syncthreads();
  V* pub_all = reinterpret_cast<V*>(scr.pub) + (size_t)gid * K::NC;
  V* xch_all = reinterpret_cast<V*>(scr.xch) + (size_t)gid * K::NC;
  uint32_t phase = 0;
  int slot = 0;
  cl.sync();  // every CTA's shared memory is initialised before any distributed-shared-memory write
  for (int64_t b = gid; b < p.batch; b += G) {
    K::decompose_one(sig + b * K::n, imfs + b * (int64_t)(p.max_imfs + 1) * K::n, count + b,
                     lens + b * p.max_imfs, iters + b * p.max_imfs, p, s, cl, tw, pub_all, xch_all, phase, slot,
                     rank, t);
  }
  cl.sync();  // no CTA exits while a partner may still write into its shared memory
}

}  // namespace cl
}  // namespace fifgpu
