// fif_streamed.cuh -- the "streamed" regime of the FIF hot path for n beyond one CTA's on-chip
// capacity (configs 2, 3 and 4: n up to 2^27, n/2 of the form 2^a 3^b 5^c).
//
// The spectrum X (digit-reversed multi-level order, below) and the time-domain remainder R live in
// HBM (R in the trend slot of d_imfs); the IMF slot being produced doubles as the inverse FFT's work
// buffer.  Every IMF is a fixed, short sequence of stream-ordered kernels over the whole batch, with
// per-signal state (k, L, N, M, active) in device arrays, so fif_decompose never synchronises.
//
// Multi-level FFT over NC = n/2 complex points z_m = x_2m + i x_2m+1 ("U^T s is the DFT
// of s ... FFT"): NC = F_0 F_1 ... F_{L-1}; digit i has stride S_i = F_{i+1}...F_{L-1}.  Forward pass
// i (i = 0..L-1) does, for every block and every lower index s < S_i, a length-F_i DFT over the digit
// (stride S_i) and multiplies element (k_i, s) by e^{-2 pi i s k_i/(F_i S_i)}; the result sits at
// position sum k_i S_i and holds bin sum k_i F_0..F_{i-1} ("digit reversed").  The inverse runs the
// passes backwards (conjugate twiddle first, then the IDFT) and ends in natural order.  The last
// level (S = 1) is a contiguous row; rows come in Hermitian mirror pairs (bin k of row base+P t pairs
// with bin NC-k at row P-base, element F-1-t), so the real-FFT post-processing (forward) and the
// damping + real-IFFT pre-processing (inverse), which couple X_k and X_{NC-k}, fuse into the row pass.
//
// Steps (same readings as fif_resident.cuh):
//   a1  k_col<FWD_FIRST> .. k_rows_fwd: forward FFT + Hermitian post-processing
//   a2  extrema: per-segment monoid partials written by the level-0 passes, folded by
//       k_fold (ordered, two levels)                                                   (A4)
//   a3  L from k in k_fold (A1, A3, A8: floor(fl(fl(xi n)/k)) in IEEE fp64)
//   a4  w_hat_k = [sin(pi r/n)/(L sin(pi k/n))]^4, sines from a two-level table of
//       e^{i pi j/n} (exact integer reduction of r = L k mod n)
//   a5  k_probe: fp64 Parseval sums at N = cap, then K-ary fp64 rounds if SD(cap) <= delta
//       (SD monotone in N, P7); the last CTA of each signal decides
//   a6  k_rows_inv: a^N damping, X <- (1-a^N) X, pre-processing, row IDFTs; middle
//       passes; k_col<INV_LAST>: level-0 IDFT, IMF store, R -= IMF, extrema partials
//   a7  k_fold bookkeeping (l_m, N_m, M), k_final: trend in slot M, zero fill
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fif_resident.cuh"

namespace fifgpu {
namespace st {

constexpr int kMaxLev = 4;
constexpr int kMaxPass = 16;
constexpr int kProbes = 15;  // K-ary search: probes per round
constexpr int kThreads = 256;
constexpr int kNW = kThreads / 32;
#ifndef FIF_COL_THREADS
#define FIF_COL_THREADS 256
#endif
constexpr int kColThreads = FIF_COL_THREADS;  // block size of the column passes
#ifndef FIF_PROBE1_MINB
#define FIF_PROBE1_MINB 2  // K-ary probe kernel: 30 fp64 accumulators per thread -> a 128-register budget
#endif
#ifndef FIF_ST_MINB
#define FIF_ST_MINB 3  // resident CTAs per SM the heavy streamed kernels are register-budgeted for
#endif
#ifndef FIF_ROWS_MINB
#define FIF_ROWS_MINB 2  // the inverse row kernel: 3 x 32 KiB of shared memory (two staging buffers + one FFT buffer)
#endif

struct Level {
  int F;          // sub-FFT length of this digit
  int C;          // columns (consecutive lower indices s) per tile; 2 rows (a mirror pair) for the row level
  int pitch;      // shared-memory column pitch (complex elements)
  int np;         // radix passes of the length-F FFT
  int rad[kMaxPass];
  int twoff;      // offset of e^{-2 pi i j/F} (j < F) in the Stockham twiddle table
  int64_t S;      // stride of the digit
  int64_t A;      // blocks = NC / (F S)
  int64_t E2;     // 2n / (F S): E-table index step of the inter-level twiddle
  int64_t tiles;  // tiles per signal = A S / C (column levels)
  int cs;         // log2(C) when C is a power of two, else -1
  int swz;        // 1: XOR-swizzled columns (F a multiple of the 128-byte row), pitch = F
};

// shared-memory slot of element i of column c: with swz, the 16-byte (8-byte) bank group of i is
// XORed with (i / row) ^ c, so column-strided (tile loads), radix-strided (Stockham stores) and
// contiguous accesses all spread over the banks
template <typename V>
__device__ __forceinline__ int sidx(int c, int i, int pitch, int swz) {
  constexpr int ROW = 128 / (int)sizeof(V), LR = sizeof(V) == 16 ? 3 : 4;
  return c * pitch + (i ^ (((i >> LR) ^ c) & ((ROW - 1) & -swz)));
}

// complex elements per tile buffer (F C <= kTile): 32 KiB of shared memory per buffer
template <typename Real> struct TileCap { static constexpr int value = 16384 / (int)sizeof(Real); };
// tile element i -> (digit f, column cc)
__device__ __forceinline__ void tile_fc(const Level& lv, int i, int& f, int& cc) {
  if (lv.cs >= 0) {
    f = i >> lv.cs;
    cc = i & (lv.C - 1);
  } else {
    f = i / lv.C;
    cc = i - f * lv.C;
  }
}

struct Geo {
  int64_t n, NC, batch;
  int L;                 // levels (>= 2)
  Level lv[kMaxLev];
  int64_t P;             // rows = NC / F_{L-1}: bin k = base + P t in a row
  int Frow;              // F_{L-1}
  int Fd[kMaxLev];       // F_i (copy of lv[i].F for the digit loops)
  int64_t Pd[kMaxLev];   // bin weight of digit i = F_0 ... F_{i-1}
  int64_t Sr[kMaxLev];   // row-index weight of digit i = S_i / F_{L-1}  (i < L-1)
  int64_t units;         // row-pair units = floor(P/2) + 1
  int64_t nseg;          // extrema segments per signal = NC / C_0 (each 2 C_0 consecutive samples)
  int64_t grp;           // segments per fold group
  int64_t ngrp;          // fold groups per signal
  int64_t nbch;          // probe chunks per signal (= units)
  int eb;                // E table split: E(j) = Eh[j >> eb] * El[j & (2^eb - 1)]
  int max_imfs, max_inner, window;
  double xi, delta2;
  int64_t sig_stride;    // reals per signal in d_imfs = (max_imfs + 1) n
  int stop;              // 0: SD rule; 1: a-priori N0 (absolute delta)
  double delta, gamma;   // delta (absolute, stop = 1); gamma-threshold (0: off)
  int mask;              // 0: extrema filter-length rule; 1: spectral-peak rule (A20)
  double* pnat;          // [B][NC+1] |X_k|^2 in natural bin order (mask = 1 only)
  const int2* utab;      // [units] rows (ra, rb) of the mirror-pair unit u (bases u and P - u)
  const int* rbase;      // [P] bin base of each row
  const int* rmir;       // [P] row holding the mirror bins of each row
};

template <typename Real>
struct Tabs {
  using V = typename Cx<Real>::V;
  const double2* Eh;  // e^{i pi (h 2^eb)/n}
  const double2* El;  // e^{i pi l/n}, l < 2^eb
  const V* Th;        // the same in Real precision (twiddles)
  const V* Tl;
  const V* tw;        // per-level Stockham twiddles
};

// per-signal control block (device)
struct Ctl {
  int32_t* k;       // extrema count of the current remainder
  int32_t* L;       // half-length of h for the current IMF
  int32_t* N;       // iteration count of the current IMF
  int32_t* M;       // IMFs done (-1: non-finite input)
  int32_t* active;  // 1 while the signal still extracts IMFs
  int32_t* search;  // 1 while the K-ary search runs
  int32_t* lo;      // search bracket: !pass(lo) (lo = 0 virtual), pass(hi)
  int32_t* hi;
  int32_t* bad;     // non-finite input seen
  int32_t* redo;    // 1: the speculative N = cap damping of this IMF is void (SD(cap) <= delta)
  double* pmax;     // [B] max_{k >= 1} |X_k|^2 (spectral-peak rule)
  int32_t* slist;   // [B] signals (wave-local) whose SD(cap) <= delta this IMF (K-ary search + redo)
  int32_t* scnt;    // [1 per wave] length of slist
  uint32_t* cnt;    // last-CTA counters
  uint32_t* segi;   // [B][nseg] packed extrema monoid of a segment's internal differences
  void* segv;       // [B][nseg][2] Real: first and last sample of the segment
  uint32_t* gi;     // [B][ngrp] packed monoid of a fold group
  void* gv;         // [B][ngrp][2] Real
  double* red;      // [B][nbch][2 kProbes] probe partial sums
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

// radix-16 DFT (natural order in and out) as 4 x 4 with the internal twiddles e^{DIR 2 pi i n2 k1/16}
template <int DIR, typename V>
__device__ __forceinline__ void dft16(V* x) {
  using S = decltype(x[0].x);
  const S c1 = (S)0.92387953251128675612818318939678829, s1 = (S)0.38268343236508977172845998403039887;
  const S h = (S)0.70710678118654752440084436210484903928;
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<DIR>(x[n2], x[4 + n2], x[8 + n2], x[12 + n2]);
  // y[n2][k1] sits at x[4 k1 + n2]; multiply by w^{n2 k1}, w = e^{DIR 2 pi i/16}
  auto tw = [&](V& v, S c, S sn) { v = V{v.x * c - (S)DIR * v.y * sn, (S)DIR * v.x * sn + v.y * c}; };
  tw(x[4 + 1], c1, s1);   // n2 = 1, k1 = 1: w^1
  tw(x[8 + 1], h, h);     // w^2
  tw(x[12 + 1], s1, c1);  // w^3
  tw(x[4 + 2], h, h);     // w^2
  x[8 + 2] = mul_i<DIR>(x[8 + 2]);  // w^4
  tw(x[12 + 2], -h, h);   // w^6
  tw(x[4 + 3], s1, c1);   // w^3
  tw(x[8 + 3], -h, h);    // w^6
  tw(x[12 + 3], -c1, -s1);  // w^9
  V y[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) y[i] = x[i];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    dft4<DIR>(y[4 * k1 + 0], y[4 * k1 + 1], y[4 * k1 + 2], y[4 * k1 + 3]);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) x[k1 + 4 * k2] = y[4 * k1 + k2];
  }
}

template <int P, int DIR, typename V>
__device__ __forceinline__ void dft_small(V* x) {
  if constexpr (P == 2) {
    const V a = cadd(x[0], x[1]), b = csub(x[0], x[1]);
    x[0] = a;
    x[1] = b;
  } else if constexpr (P == 3) {
    dft3<DIR>(x[0], x[1], x[2]);
  } else if constexpr (P == 4) {
    dft4<DIR>(x[0], x[1], x[2], x[3]);
  } else if constexpr (P == 5) {
    dft5<DIR>(x[0], x[1], x[2], x[3], x[4]);
  } else if constexpr (P == 8) {
    dft8<DIR>(x);
  } else {
    dft16<DIR>(x);
  }
}

// One Stockham pass of compile-time radix P over `cols` independent length-Ns FFTs, column c at
// offset c*pitch (slots through sidx): src[c, i] -> dst[c, j].  tw[j] = e^{-2 pi i j/Ns}.
template <int P, int DIR, typename V>
__device__ void cta_pass_t(const V* src, V* dst, int Ns, int cols, int pitch, int swz, int NS,
                           const V* __restrict__ tw) {
  const int per = Ns / P;
  const int tstride = Ns / (NS * P);
  const bool pow2 = ((Ns & (Ns - 1)) == 0) && ((NS & (NS - 1)) == 0);
  const int lper = __ffs(per) - 1;
  for (int idx = threadIdx.x; idx < cols * per; idx += blockDim.x) {
    int f, vt, k;
    if (pow2) {
      f = idx >> lper;
      vt = idx & (per - 1);
      k = vt & (NS - 1);
    } else {
      f = idx / per;
      vt = idx - f * per;
      k = vt % NS;
    }
    V x[P];
#pragma unroll
    for (int r = 0; r < P; ++r) x[r] = src[sidx<V>(f, vt + r * per, pitch, swz)];
    if (NS > 1) {
      const int kt = k * tstride;
#pragma unroll
      for (int r = 1; r < P; ++r) {
        V t = tw[r * kt];  // (global or shared)
        if (DIR > 0) t.y = -t.y;
        x[r] = cmul(x[r], t);
      }
    }
    dft_small<P, DIR>(x);
    const int j0 = (vt - k) * P + k;  // (vt / NS) NS P + k
#pragma unroll
    for (int r = 0; r < P; ++r) dst[sidx<V>(f, j0 + r * NS, pitch, swz)] = x[r];
  }
}
template <int DIR, typename V, int MAXR = 16>
__device__ __forceinline__ void cta_pass(const V* src, V* dst, int Ns, int cols, int pitch, int swz, int p, int NS,
                                         const V* __restrict__ tw) {
  switch (p) {
    case 2: cta_pass_t<2, DIR>(src, dst, Ns, cols, pitch, swz, NS, tw); break;
    case 3: cta_pass_t<3, DIR>(src, dst, Ns, cols, pitch, swz, NS, tw); break;
    case 4: cta_pass_t<4, DIR>(src, dst, Ns, cols, pitch, swz, NS, tw); break;
    case 5: cta_pass_t<5, DIR>(src, dst, Ns, cols, pitch, swz, NS, tw); break;
    case 8: cta_pass_t<8, DIR>(src, dst, Ns, cols, pitch, swz, NS, tw); break;
    default:
      if constexpr (MAXR >= 16) cta_pass_t<16, DIR>(src, dst, Ns, cols, pitch, swz, NS, tw);
      break;
  }
}

// All passes of a level; a holds the input, returns the buffer holding the output (a or b).  MAXR = 8:
// the level's schedule has no radix-16 pass (fp64 geometries, radices(..., 8)), so its 64-register
// butterfly is not compiled into the caller.
template <int DIR, typename V, int MAXR = 16>
__device__ V* cta_fft(V* a, V* b, const Level& lv, int cols, const V* __restrict__ tw) {
  int NS = 1;
  for (int ps = 0; ps < lv.np; ++ps) {
    __syncthreads();
    cta_pass<DIR, V, MAXR>(a, b, lv.F, cols, lv.pitch, lv.swz, lv.rad[ps], NS, tw + lv.twoff);
    NS *= lv.rad[ps];
    V* t = a; a = b; b = t;
  }
  __syncthreads();
  return a;
}

// The same passes with the transform length, a radix schedule and the swizzled pitch known at compile
// time: constant index math.
// the twiddles of the thread's first butterfly of a pass (they depend on neither the data nor the previous
// pass): loaded BEFORE the pass's barrier, so the table latency overlaps the barrier wait
template <int P, int DIR, typename V, int F, int NS>
__device__ __forceinline__ void pass_tw_pre(V (&t)[P], const V* __restrict__ tw) {
  if constexpr (NS > 1) {
    constexpr int per = F / P, tstride = F / (NS * P);
    const int kt = ((int)(threadIdx.x % per) % NS) * tstride;
#pragma unroll
    for (int r = 1; r < P; ++r) t[r] = tw[r * kt];
  }
}
template <int P, int DIR, typename V, int F, int NS, int PITCH = F, int SWZ = 1, bool PRE = false>
__device__ __forceinline__ void cta_pass_c(const V* src, V* dst, int cols, const V* __restrict__ tw,
                                           const V (&tpre)[P]) {
  constexpr int per = F / P, tstride = F / (NS * P);
  for (int idx = threadIdx.x; idx < cols * per; idx += blockDim.x) {
    const int f = idx / per, vt = idx % per, k = vt % NS;
    V x[P];
#pragma unroll
    for (int r = 0; r < P; ++r) x[r] = src[sidx<V>(f, vt + r * per, PITCH, SWZ)];
    if constexpr (NS > 1) {
      const int kt = k * tstride;
      const bool first = PRE && idx == (int)threadIdx.x;
#pragma unroll
      for (int r = 1; r < P; ++r) {
        V t = first ? tpre[r] : tw[r * kt];
        if (DIR > 0) t.y = -t.y;
        x[r] = cmul(x[r], t);
      }
    }
    dft_small<P, DIR>(x);
    const int j0 = (vt - k) * P + k;
#pragma unroll
    for (int r = 0; r < P; ++r) dst[sidx<V>(f, j0 + r * NS, PITCH, SWZ)] = x[r];
  }
}
// PRE: twiddles from global memory, prefetched ahead of each pass's barrier (the row passes); the column
// passes read theirs from shared memory and keep the registers
template <int DIR, typename V, int F, int NS, int P, int... Rest>
__device__ __forceinline__ V* cta_fft_c_pre(V* a, V* b, int cols, const V* __restrict__ tw) {
  V tpre[P];
  pass_tw_pre<P, DIR, V, F, NS>(tpre, tw);
  __syncthreads();
  cta_pass_c<P, DIR, V, F, NS, F, 1, true>(a, b, cols, tw, tpre);
  if constexpr (sizeof...(Rest) == 0) {
    __syncthreads();
    return b;
  } else {
    return cta_fft_c_pre<DIR, V, F, NS * P, Rest...>(b, a, cols, tw);
  }
}
template <int DIR, typename V, int F, int NS, int P, int... Rest>
__device__ __forceinline__ V* cta_fft_c(V* a, V* b, int cols, const V* __restrict__ tw) {
  V tpre[P];
  __syncthreads();
  cta_pass_c<P, DIR, V, F, NS>(a, b, cols, tw, tpre);
  if constexpr (sizeof...(Rest) == 0) {
    __syncthreads();
    return b;
  } else {
    return cta_fft_c<DIR, V, F, NS * P, Rest...>(b, a, cols, tw);
  }
}
// the same for an unswizzled (odd-pitch) level: the mixed-radix column lengths
template <int DIR, typename V, int F, int NS, int P, int... Rest>
__device__ __forceinline__ V* cta_fft_c_odd(V* a, V* b, int cols, const V* __restrict__ tw) {
  V tpre[P];
  __syncthreads();
  cta_pass_c<P, DIR, V, F, NS, F + 1, 0>(a, b, cols, tw, tpre);
  if constexpr (sizeof...(Rest) == 0) {
    __syncthreads();
    return b;
  } else {
    return cta_fft_c_odd<DIR, V, F, NS * P, Rest...>(b, a, cols, tw);
  }
}
// Row-major tiles (the column passes whose tiles are staged by cp.async.bulk, one copy per tile row): element
// (column c, digit i) at i * cols + c.  Column fastest over the threads, so the lanes of a warp read and write
// contiguous row segments (conflict-free without a swizzle) and share their twiddle.
template <int P, int DIR, typename V, int F, int NS>
__device__ __forceinline__ void cta_pass_rm(const V* src, V* dst, int cols, const V* __restrict__ tw) {
  constexpr int per = F / P, tstride = F / (NS * P);
  // (power-of-two tile widths -- every benchmark geometry -- split the index by a shift, not a division)
  const int csh = (cols & (cols - 1)) == 0 ? 31 - __clz(cols) : -1;
  for (int idx = threadIdx.x; idx < cols * per; idx += blockDim.x) {
    const int vt = csh >= 0 ? idx >> csh : idx / cols, c = idx - vt * cols, k = vt % NS;
    V x[P];
#pragma unroll
    for (int r = 0; r < P; ++r) x[r] = src[(vt + r * per) * cols + c];
    if constexpr (NS > 1) {
      const int kt = k * tstride;
#pragma unroll
      for (int r = 1; r < P; ++r) {
        V t = tw[r * kt];
        if (DIR > 0) t.y = -t.y;
        x[r] = cmul(x[r], t);
      }
    }
    dft_small<P, DIR>(x);
    const int j0 = (vt - k) * P + k;
#pragma unroll
    for (int r = 0; r < P; ++r) dst[(j0 + r * NS) * cols + c] = x[r];
  }
}
template <int DIR, typename V, int F, int NS, int P, int... Rest>
__device__ __forceinline__ V* cta_fft_rm(V* a, V* b, int cols, const V* __restrict__ tw) {
  __syncthreads();
  cta_pass_rm<P, DIR, V, F, NS>(a, b, cols, tw);
  if constexpr (sizeof...(Rest) == 0) {
    __syncthreads();
    return b;
  } else {
    return cta_fft_rm<DIR, V, F, NS * P, Rest...>(b, a, cols, tw);
  }
}
template <int F, int... R>
__device__ __forceinline__ bool sched_is(const Level& lv) {
  constexpr int r[] = {R...};
  if (lv.F != F || !lv.swz || lv.pitch != F || lv.np != (int)sizeof...(R)) return false;
  for (int i = 0; i < (int)sizeof...(R); ++i)
    if (lv.rad[i] != r[i]) return false;
  return true;
}
// Row transforms: the compile-time path for the full-length rows (every benchmark configuration), the
// generic passes otherwise.
// Row transforms.  RS selects, per kernel instance, ONE path (the host picks it: row_schedule() in
// fif_st.cu): 1 = the full-length rows of every benchmark geometry at compile time (fp64 1024 = 2 8 8 8,
// radix <= 8 so the 64-register radix-16 butterfly is never compiled into an fp64 kernel; fp32
// 2048 = 8 16 16), 0 = the generic passes.
template <int DIR, typename V, int RS>
__device__ __forceinline__ V* row_fft(V* a, V* b, const Level& lv, int cols, const V* __restrict__ tw) {
  if constexpr (RS == 1 && sizeof(V) == 16) return cta_fft_c_pre<DIR, V, 1024, 1, 2, 8, 8, 8>(a, b, cols, tw + lv.twoff);
  else if constexpr (RS == 1) return cta_fft_c_pre<DIR, V, 2048, 1, 8, 16, 16>(a, b, cols, tw + lv.twoff);
  else return cta_fft<DIR, V, sizeof(V) == 16 ? 8 : 16>(a, b, lv, cols, tw);
}
// Column transforms.  CS selects, per kernel instance, ONE transform path (the host picks it from the
// level: col_schedule() in fif_st.cu), so each k_col instance carries only the code it runs:
//   0 generic passes (fp64: radix <= 8), 1-4 fp32 F = 32 / 64 / 128 / 256, 5-8 fp64 F = 128 / 256 / 32 / 64,
//   9-10 fp32 F = 12 / 20 (unswizzled, pitch F + 1), 11-12 the row lengths (distributed passes),
// each with the radices() schedule and the swizzled pitch F at compile time.  tw: the level's twiddles.
template <int DIR, typename V, int CS>
__device__ __forceinline__ V* col_fft(V* a, V* b, const Level& lv, int cols, const V* __restrict__ tw) {
  if constexpr (CS == 1) return cta_fft_c<DIR, V, 32, 1, 8, 4>(a, b, cols, tw);
  else if constexpr (CS == 2) return cta_fft_c<DIR, V, 64, 1, 4, 16>(a, b, cols, tw);
  else if constexpr (CS == 3) return cta_fft_c<DIR, V, 128, 1, 8, 16>(a, b, cols, tw);
  else if constexpr (CS == 4) return cta_fft_c<DIR, V, 256, 1, 16, 16>(a, b, cols, tw);
  else if constexpr (CS == 5) return cta_fft_c<DIR, V, 128, 1, 2, 8, 8>(a, b, cols, tw);
  else if constexpr (CS == 6) return cta_fft_c<DIR, V, 256, 1, 4, 8, 8>(a, b, cols, tw);
  else if constexpr (CS == 7) return cta_fft_c<DIR, V, 32, 1, 4, 8>(a, b, cols, tw);
  else if constexpr (CS == 8) return cta_fft_c<DIR, V, 64, 1, 8, 8>(a, b, cols, tw);
  else if constexpr (CS == 9) return cta_fft_c_odd<DIR, V, 12, 1, 4, 3>(a, b, cols, tw);
  else if constexpr (CS == 10) return cta_fft_c_odd<DIR, V, 20, 1, 4, 5>(a, b, cols, tw);
  else if constexpr (CS == 11) return cta_fft_c<DIR, V, 1024, 1, 2, 8, 8, 8>(a, b, cols, tw);
  else if constexpr (CS == 12) return cta_fft_c<DIR, V, 2048, 1, 8, 16, 16>(a, b, cols, tw);
  // 21-30: CS - 20 on row-major tiles (k_col with bulk-copy staging)
  else if constexpr (CS == 21) return cta_fft_rm<DIR, V, 32, 1, 8, 4>(a, b, cols, tw);
  else if constexpr (CS == 22) return cta_fft_rm<DIR, V, 64, 1, 4, 16>(a, b, cols, tw);
  else if constexpr (CS == 23) return cta_fft_rm<DIR, V, 128, 1, 8, 16>(a, b, cols, tw);
  else if constexpr (CS == 24) return cta_fft_rm<DIR, V, 256, 1, 16, 16>(a, b, cols, tw);
  else if constexpr (CS == 25) return cta_fft_rm<DIR, V, 128, 1, 2, 8, 8>(a, b, cols, tw);
  else if constexpr (CS == 26) return cta_fft_rm<DIR, V, 256, 1, 4, 8, 8>(a, b, cols, tw);
  else if constexpr (CS == 27) return cta_fft_rm<DIR, V, 32, 1, 4, 8>(a, b, cols, tw);
  else if constexpr (CS == 28) return cta_fft_rm<DIR, V, 64, 1, 8, 8>(a, b, cols, tw);
  else if constexpr (CS == 29) return cta_fft_rm<DIR, V, 12, 1, 4, 3>(a, b, cols, tw);
  else if constexpr (CS == 30) return cta_fft_rm<DIR, V, 20, 1, 4, 5>(a, b, cols, tw);
  else return cta_fft<DIR, V, sizeof(V) == 16 ? 8 : 16>(a, b, lv, cols, tw);
}

// ------------------------------------------------------------------ tables
// E(j) = e^{i pi j/n}, 0 <= j <= 2n, from the two-level table (one complex product)
template <typename I = int64_t>
__device__ __forceinline__ double2 E64(const double2* __restrict__ Eh, const double2* __restrict__ El, int eb, I j) {
  return cmul(__ldg(Eh + (j >> eb)), __ldg(El + (j & (((I)1 << eb) - 1))));
}
// sin(pi j/n) for 0 <= j <= n/2: both table angles lie in the first quadrant, so the imaginary part
// of the product is a sum of two non-negative terms (relative error ~2 ulp)
__device__ __forceinline__ double sin_n(const double2* __restrict__ Eh, const double2* __restrict__ El, int eb,
                                        int64_t j) {
  const double2 h = __ldg(Eh + (j >> eb)), l = __ldg(El + (j & ((1LL << eb) - 1)));
  return h.x * l.y + h.y * l.x;
}
template <typename Real>
__device__ __forceinline__ typename Cx<Real>::V Er(const Tabs<Real>& tb, int eb, int64_t j) {
  return cmul(__ldg(tb.Th + (j >> eb)), __ldg(tb.Tl + (j & ((1LL << eb) - 1))));
}

// (E2 x) mod 2n for an inter-level twiddle index: E2 (x mod F S) = (E2 x) mod 2n since E2 F S = 2n, and E(j)
// has period 2n -- a mask for power-of-two n instead of a 64-bit division per tile or element
__device__ __forceinline__ int64_t mod2n(const Geo& g, int64_t x) {
  const int64_t m = 2 * g.n;
  return (g.n & (g.n - 1)) == 0 ? (x & (m - 1)) : x % m;
}
// a4: w_hat_k for 0 <= k <= n/2: r = min(L k mod n, n - L k mod n)
template <typename Real>
__device__ __forceinline__ double what_tab(const Geo& g, const Tabs<Real>& tb, int L, int64_t k) {
  if (k == 0) return 1.0;
  const int64_t m = ((int64_t)L * k) % g.n;
  const int64_t r = m < g.n - m ? m : g.n - m;
  const double s = sin_n(tb.Eh, tb.El, g.eb, r) / ((double)L * sin_n(tb.Eh, tb.El, g.eb, k));
  const double s2 = s * s;
  return s2 * s2;
}
// x mod n for 0 <= x < 2^53 (one fp64 multiply by 1/n, one correction step)
__device__ __forceinline__ int64_t mod_n(int64_t x, int64_t n, double invn) {
  const int64_t q = (int64_t)((double)x * invn);
  int64_t m = x - q * n;
  if (m < 0) m += n;
  else if (m >= n) m -= n;
  return m;
}
// a4 for a Hermitian pair (k, NC - k), 0 <= k < NC, given mk = L k mod n: one division and two
// table products for both bins.  sin(pi (NC-k)/n) = cos(pi k/n); L (NC - k) = L NC - L k with
// L NC = 0 (L even) or NC (L odd) mod n, so sin(pi r_{NC-k}/n) = sin(pi mk/n) (L even) or
// |cos(pi mk/n)| (L odd).  A cosine near zero carries a larger relative error, but it then belongs
// to a bin whose w_hat is tiny or whose a^N vanishes, so the absolute error of a^N stays at
// rounding level (|d a^N| <= N a^{N-1} |d w| <= |d w / w| / e).  Returns e^{i pi k/n} in Ek.
template <typename Real, typename I = int64_t>
__device__ __forceinline__ void what_pair_m(const Geo& g, const Tabs<Real>& tb, int L, I k, I mk,
                                            double& wk, double& wm, double2& Ek) {
  const I rk = mk <= (I)g.NC ? mk : (I)g.n - mk;
  Ek = E64(tb.Eh, tb.El, g.eb, k);                 // (cos, sin)(pi k/n), first quadrant
  const double2 Er_ = E64(tb.Eh, tb.El, g.eb, rk);  // (cos, sin)(pi rk/n), first quadrant
  const double nk = Er_.y, nm = (L & 1) ? fabs(Er_.x) : Er_.y;
  const double dk = Ek.y, dm = Ek.x;
  const double Ld = (double)L;
  double sk, sm;
  if (k == 0) {
    sk = 1.0;
    sm = nm / (Ld * dm);
  } else {
    const double inv = 1.0 / (Ld * Ld * dk * dm);
    sk = nk * Ld * dm * inv;
    sm = nm * Ld * dk * inv;
  }
  sk *= sk;
  sm *= sm;
  wk = sk * sk;
  wm = sm * sm;
}
// the same from k alone
template <typename Real>
__device__ __forceinline__ void what_pair(const Geo& g, const Tabs<Real>& tb, int L, double invn, int64_t k,
                                          double& wk, double& wm) {
  double2 Ek;
  what_pair_m(g, tb, L, k, mod_n((int64_t)L * k, g.n, invn), wk, wm, Ek);
}
template <int E>
__device__ __forceinline__ double upow_c(double a) {
  double e[1], x[1] = {a};
  upow_ct<E, 1, double>(e, x);
  return e[0];
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

// fp32 plans (reading A14): the damping powers and the probe terms in fp32.  a^m = 2^(m log2(1 - w)) through
// the SFU; log2(1 - w) from the series -(w + w^2/2 + ... + w^7/7) log2(e) for w < 1/16 (relative error
// ~1e-7 of w, truncation < w^7/8), lg2.approx(1 - w) above (absolute error ~2^-22: relative error of a^m
// m 2^-22 ln 2, on values a^m <= (15/16)^m that are then tiny).  w >= 1 (rounding) gives log2 0 = -inf, a^m = 0.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float log2_1m(float w) {
  float p = fmaf(w, 1.f / 7.f, 1.f / 6.f);
  p = fmaf(w, p, 0.2f);
  p = fmaf(w, p, 0.25f);
  p = fmaf(w, p, 1.f / 3.f);
  p = fmaf(w, p, 0.5f);
  p = fmaf(w, p, 1.f);
  const float ser = -1.44269504088896341f * w * p;
  float lg;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(fmaxf(1.f - w, 0.f)));
  return w < 0.0625f ? ser : lg;
}
__device__ __forceinline__ float pow_l2(float l2, int m) { return m > 0 ? ex2_approx((float)m * l2) : 1.f; }

// row index (position / F_{L-1}) of the row whose bins are base + P t, and back
__device__ __forceinline__ int64_t row_of_base(const Geo& g, int64_t base) {
  int64_t r = 0;
#pragma unroll
  for (int i = 0; i < kMaxLev - 1; ++i)
    if (i < g.L - 1) r += ((base / g.Pd[i]) % g.Fd[i]) * g.Sr[i];
  return r;
}
__device__ __forceinline__ int64_t base_of_row(const Geo& g, int64_t row) {
  int64_t b = 0;
#pragma unroll
  for (int i = 0; i < kMaxLev - 1; ++i)
    if (i < g.L - 1) b += ((row / g.Sr[i]) % g.Fd[i]) * g.Pd[i];
  return b;
}

// ------------------------------------------------------------------ a2 extrema monoid
// Over a sequence of differences: f = first nonzero sign, l = last nonzero sign, c = sign changes
// among the nonzero ones (zero differences dropped: plateau collapse, reading A4).
struct Mono {
  int f, l, c;
};
__device__ __forceinline__ Mono mcomb(Mono a, Mono b) {
  return Mono{a.f ? a.f : b.f, b.l ? b.l : a.l, a.c + b.c + ((a.l && b.f && a.l != b.f) ? 1 : 0)};
}
template <typename Real>
__device__ __forceinline__ Mono mdiff(Real d) {
  const int s = d > (Real)0 ? 1 : (d < (Real)0 ? -1 : 0);
  return Mono{s, s, 0};
}
__device__ __forceinline__ uint32_t mpack(Mono m) {
  return (uint32_t)(m.f + 1) | ((uint32_t)(m.l + 1) << 2) | ((uint32_t)m.c << 4);
}
__device__ __forceinline__ Mono munpack(uint32_t u) {
  return Mono{(int)(u & 3) - 1, (int)((u >> 2) & 3) - 1, (int)(u >> 4)};
}
// ordered warp reduction: lane 0 receives lanes 0..31 combined in lane order
__device__ __forceinline__ Mono warp_mono(Mono m) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Mono o;
    o.f = __shfl_down_sync(0xffffffffu, m.f, off);
    o.l = __shfl_down_sync(0xffffffffu, m.l, off);
    o.c = __shfl_down_sync(0xffffffffu, m.c, off);
    if ((lane & (2 * off - 1)) == 0 && lane + off < 32) m = mcomb(m, o);
  }
  return m;
}
// ordered block reduction; the result is valid in thread 0
__device__ __forceinline__ Mono block_mono(Mono m, Mono* sm) {
  m = warp_mono(m);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    Mono r = sm[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = mcomb(r, sm[w]);
    m = r;
  }
  return m;
}

// Segment partials of a level-0 tile held in shared memory as complex pairs: segment f consists of
// the 2C reals of columns c = 0..C-1 (element (c, f) at slot sidx(c, f)); one warp per segment.
// Fast path (no zero difference in the segment): lane l owns the differences starting at its reals,
// the last one reaching into lane l+1's first real; sign changes = popc of adjacent sign-bit XORs
// inside a lane + the lane-boundary transitions, summed with a warp reduction.  A zero difference
// anywhere in the segment (plateau collapse, reading A4) switches the warp to the exact ordered
// monoid fold.
template <typename Real, bool RM = false>
__device__ void tile_segments(const typename Cx<Real>::V* buf, const Level& lv, int64_t seg0, int64_t segstep,
                              uint32_t* __restrict__ segi, Real* __restrict__ segv) {
  using V = typename Cx<Real>::V;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nr = 2 * lv.C;           // reals per segment
  const int per = (nr + 31) / 32;    // reals per lane (the fast path needs <= 64)
  const int j0 = lane * per, j1 = min(j0 + per, nr);
  for (int f = warp; f < lv.F; f += nw) {
    auto x_at = [&](int j) -> Real {
      const V v = RM ? buf[f * lv.C + (j >> 1)] : buf[sidx<V>(j >> 1, f, lv.pitch, lv.swz)];
      return (j & 1) ? v.y : v.x;
    };
    // this lane's reals and the first real of the next lane
    Real first = (Real)0, prev = (Real)0;
    uint64_t bits = 0;
    int nd = 0;
    bool zero = per > 64;
    if (j0 < j1 && !zero) {
      first = x_at(j0);
      prev = first;
      for (int j = j0 + 1; j < j1; ++j) {
        const Real x = x_at(j);
        const Real d = x - prev;
        zero |= (d == (Real)0);
        bits |= (uint64_t)(d < (Real)0) << nd;
        ++nd;
        prev = x;
      }
    }
    const Real nxt = __shfl_down_sync(0xffffffffu, first, 1);
    if (j0 < j1 && j1 < nr && per <= 64) {  // the difference into the next lane's first real
      const Real d = nxt - prev;
      zero |= (d == (Real)0);
      bits |= (uint64_t)(d < (Real)0) << nd;
      ++nd;
    }
    Mono m;
    if (!__any_sync(0xffffffffu, zero)) {
      const int inner = nd > 1 ? __popcll((bits ^ (bits >> 1)) & ((nd - 1 >= 64) ? ~0ull : ((1ull << (nd - 1)) - 1ull))) : 0;
      const int fb = nd ? (int)(bits & 1ull) : -1, lb = nd ? (int)((bits >> (nd - 1)) & 1ull) : -1;
      const int fnext = __shfl_down_sync(0xffffffffu, fb, 1);
      const int edge = (nd && lane < 31 && fnext >= 0 && fnext != lb) ? 1 : 0;
      const int total = __reduce_add_sync(0xffffffffu, inner + edge);
      // first / last nonzero signs of the segment (no zeros: the first and the last difference)
      const int f0 = __shfl_sync(0xffffffffu, fb, 0);
      const int lastLane = (nr - 2) / per;  // owner of the last difference (reals nr-2 -> nr-1)
      const int l0 = __shfl_sync(0xffffffffu, lb, lastLane);
      m = Mono{f0 < 0 ? 0 : (f0 ? -1 : 1), l0 < 0 ? 0 : (l0 ? -1 : 1), total};
    } else {
      m = Mono{0, 0, 0};
      const int nd2 = nr - 1, q = (nd2 + 31) / 32;
      const int d0 = lane * q, d1 = min(d0 + q, nd2);
      if (d0 < d1) {
        Real pv = x_at(d0);
        for (int j = d0; j < d1; ++j) {
          const Real x = x_at(j + 1);
          m = mcomb(m, mdiff<Real>(x - pv));
          pv = x;
        }
      }
      m = warp_mono(m);
    }
    if (lane == 0) {
      const int64_t sg = seg0 + (int64_t)f * segstep;
      segi[sg] = mpack(m);
      segv[2 * sg] = x_at(0);
      segv[2 * sg + 1] = x_at(nr - 1);
    }
  }
}

// Thread-chunk variant of tile_segments: the tps threads t = f + F q (q = 0..tps-1; tps the largest power
// of two dividing 2C with F tps <= blockDim) of segment f own its consecutive chunks q of R = 2C / tps reals -- the lanes of a warp read the same
// column at consecutive rows, conflict-free -- each reduces its chunk (sign bits, one popc; the exact
// rule when a difference is zero) including the difference into the next chunk, and thread f folds the
// tps packed monoids in order.  Returns false (nothing written) when the tile shape does not allow it.
template <typename Real>
__device__ bool tile_segments_thr(const typename Cx<Real>::V* buf, const Level& lv, int64_t seg0, int64_t segstep,
                                  uint32_t* __restrict__ segi, Real* __restrict__ segv) {
  using V = typename Cx<Real>::V;
  __shared__ uint32_t pks[kColThreads];
  const int F = lv.F, nr = 2 * lv.C, nt = (int)blockDim.x;
  if (nt > kColThreads || F > nt) return false;
  int tps = 1;  // chunks per segment: the largest power of two dividing nr with F tps <= blockDim
  while (2 * tps * F <= nt && nr % (2 * tps) == 0) tps *= 2;
  const int R = nr / tps;
  if (R > 64 || (R & 1)) return false;
  const int t = threadIdx.x, f = t % F, q = t / F, c0 = q * (R >> 1);
  const bool active = t < F * tps;  // the remaining threads only take part in the barrier
  const bool last = q == tps - 1;
  uint64_t bits = 0;
  int nd = 0;
  bool zero = false;
  Real prev;
  if (active) {
    {
      const V v = buf[sidx<V>(c0, f, lv.pitch, lv.swz)];
      const Real d = v.y - v.x;
      zero |= d == (Real)0;
      bits |= (uint64_t)(d < (Real)0);
      nd = 1;
      prev = v.y;
    }
    for (int c = c0 + 1; c < c0 + R / 2; ++c) {
      const V v = buf[sidx<V>(c, f, lv.pitch, lv.swz)];
      const Real d0 = v.x - prev, d1 = v.y - v.x;
      zero |= (d0 == (Real)0) | (d1 == (Real)0);
      bits |= ((uint64_t)(d0 < (Real)0) << nd) | ((uint64_t)(d1 < (Real)0) << (nd + 1));
      nd += 2;
      prev = v.y;
    }
    Real nxt = (Real)0;
    if (!last) {  // the difference into the next chunk's first real
      nxt = buf[sidx<V>(c0 + R / 2, f, lv.pitch, lv.swz)].x;
      const Real d = nxt - prev;
      zero |= d == (Real)0;
      bits |= (uint64_t)(d < (Real)0) << nd;
      ++nd;
    }
    Mono m;
    if (!zero) {
      const int cnt = nd > 1 ? __popcll((bits ^ (bits >> 1)) & ((1ull << (nd - 1)) - 1ull)) : 0;
      m = Mono{(bits & 1ull) ? -1 : 1, ((bits >> (nd - 1)) & 1ull) ? -1 : 1, cnt};
    } else {  // zero differences are dropped (A4): the exact sequential rule over this chunk
      m = Mono{0, 0, 0};
      Real pv = buf[sidx<V>(c0, f, lv.pitch, lv.swz)].x;
      for (int j = 2 * c0 + 1; j < 2 * c0 + R; ++j) {
        const V v = buf[sidx<V>(j >> 1, f, lv.pitch, lv.swz)];
        const Real x = (j & 1) ? v.y : v.x;
        m = mcomb(m, mdiff<Real>(x - pv));
        pv = x;
      }
      if (!last) m = mcomb(m, mdiff<Real>(nxt - pv));
    }
    pks[t] = mpack(m);
  }
  __syncthreads();
  if (q == 0) {
    Mono acc = munpack(pks[f]);
    for (int qq = 1; qq < tps; ++qq) acc = mcomb(acc, munpack(pks[f + qq * F]));
    const int64_t sg = seg0 + (int64_t)f * segstep;
    segi[sg] = mpack(acc);
    segv[2 * sg] = buf[sidx<V>(0, f, lv.pitch, lv.swz)].x;
    segv[2 * sg + 1] = buf[sidx<V>(lv.C - 1, f, lv.pitch, lv.swz)].y;
  }
  return true;
}

// Ordered fold of items [i0, i1) (monoid + first/last value), boundary differences between
// consecutive items included (those before i0 are not).  Result in thread 0: monoid, first, last.
template <typename Real>
__device__ Mono fold_items(const uint32_t* __restrict__ mi, const Real* __restrict__ mv, int64_t i0, int64_t i1,
                           Mono* sm) {
  const int64_t len = i1 - i0, per = (len + blockDim.x - 1) / blockDim.x;
  const int64_t a0 = i0 + (int64_t)threadIdx.x * per, a1 = min(a0 + per, i1);
  Mono acc{0, 0, 0};
  if (a0 < a1) {
    Real prev = a0 > i0 ? __ldcg(mv + 2 * (a0 - 1) + 1) : (Real)0;
    for (int64_t s = a0; s < a1; ++s) {
      const Real first = __ldcg(mv + 2 * s), last = __ldcg(mv + 2 * s + 1);
      if (s > i0) acc = mcomb(acc, mdiff<Real>(first - prev));
      acc = mcomb(acc, munpack(__ldcg(mi + s)));
      prev = last;
    }
  }
  return block_mono(acc, sm);
}

__device__ __forceinline__ int filter_half_length(const Geo& g, int k) {
  // PAPER.md:81 l = 2 floor(nu N / k) with reading A1 (h half-support L = floor(xi n/k)), A3 clamp,
  // A8 IEEE evaluation (no contraction)
  const double tq = __dmul_rn(g.xi, (double)g.n);
  const double u = __ddiv_rn(tq, (double)k);
  long long q = (long long)floor(u);
  long long L = g.window ? 2 * q : q;
  const long long Lmax = (g.n - 1) / 4;
  if (L < 2) L = 2;
  if (L > Lmax) L = Lmax;
  return (int)L;
}

// ------------------------------------------------------------------ init
static __global__ void k_init(const __grid_constant__ Geo g, const __grid_constant__ Ctl c) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < g.batch;
       b += (int64_t)gridDim.x * blockDim.x) {
    c.M[b] = 0;
    c.bad[b] = 0;
    c.active[b] = 1;
    c.search[b] = 0;
    c.redo[b] = 0;
    c.cnt[b] = 0;
  }
}

// ------------------------------------------------------------------ bulk copies (TMA engine)
// cp.async.bulk global -> shared with mbarrier completion (transaction bytes): one instruction moves a whole
// contiguous row; the copy engine runs it while the CTA transforms the previous unit.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// cp.async.bulk.tensor: one instruction lands a whole F x C tile (a 3-D box {C, F, 1} of the tensor map
// {lower index s, digit row a F + f, signal / IMF slot}) in row-major order, completion on the mbarrier
__device__ __forceinline__ void tensor_g2s(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
      ::"r"(smem_u32(dst)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// generic-proxy accesses to a buffer (ordered by a barrier) before the async proxy refills it
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// ------------------------------------------------------------------ column passes
enum { PASS_MID = 0, PASS_FWD_FIRST = 1, PASS_INV_LAST = 2 };

// cp.async (Ampere+ LDGSTS) helpers: global -> shared without registers, completion by groups
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(d), "l"(gsrc), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Tile = C consecutive lower indices s x the F digit values, of block a.  DIR -1: forward (DFT, then
// the level's twiddle at the store), +1: inverse (IDFT; the input already carries this level's
// conjugate twiddle, applied by the producer, and the store applies the NEXT coarser level's, lvn).
// Forward passes work on X; inverse passes on the IMF slot M of the signal.  FWD_FIRST reads the
// signal (copying it to R, flagging non-finite samples, writing extrema partials of s); INV_LAST
// finishes the IMF in natural order, updates R and writes the extrema partials of the new remainder.
// Persistent CTAs, software-pipelined: the next tile streams into a third shared buffer with
// cp.async while the current one is transformed.
template <typename Real, int DIR, int KIND, int CS = 0>
__global__ void __launch_bounds__(kColThreads, 2) k_col(const __grid_constant__ Geo g, const __grid_constant__ Level lv,
                                                     const __grid_constant__ Level lvn, const Real* __restrict__ sig,
                                                     Real* __restrict__ imfs, typename Cx<Real>::V* __restrict__ X,
                                                     const __grid_constant__ Tabs<Real> tb,
                                                     const __grid_constant__ Ctl c,
                                                     const __grid_constant__ CUtensorMap tm, const int tmode) {
  using V = typename Cx<Real>::V;
  // tmode (row-major instances only): the tile is one cp.async.bulk.tensor box of the map tm (built per call by
  // the host over the source of this pass: the signals, X, or the IMF slots of d_imfs)
  // CS >= 21: row-major tiles staged by the bulk-copy engine (one cp.async.bulk per tile row, completion
  // counted in bytes on the buffer's mbarrier); else column-major XOR-swizzled tiles loaded by cp.async
  constexpr bool RMk = CS >= 21;
  extern __shared__ __align__(128) char smem_raw[];
  __shared__ __align__(8) uint64_t cmb[3];
  const size_t bufsz = (size_t)lv.C * lv.pitch;
  // tile slot of element (column cc, digit f)
  auto TI = [&](int cc, int f) { return RMk ? f * lv.C + cc : sidx<V>(cc, f, lv.pitch, lv.swz); };
  V* S[3] = {reinterpret_cast<V*>(smem_raw), reinterpret_cast<V*>(smem_raw) + bufsz,
             reinterpret_cast<V*>(smem_raw) + 2 * bufsz};
  // the level's Stockham twiddles e^{-2 pi i j/F} in shared memory (the FFT passes read 1 per point)
  V* tws = reinterpret_cast<V*>(smem_raw) + 3 * bufsz;
  for (int j = threadIdx.x; j < lv.F; j += blockDim.x) tws[j] = tb.tw[lv.twoff + j];
  Level lvs = lv;
  lvs.twoff = 0;
  const uint32_t spt = (uint32_t)(lv.S / lv.C), tiles = (uint32_t)lv.tiles;
  const uint32_t total = (uint32_t)(g.batch * lv.tiles);
  const int FC = lv.F * lv.C;
  constexpr int U = TileCap<Real>::value / kColThreads;
  auto active = [&](uint32_t t) { return KIND == PASS_FWD_FIRST || c.active[t / tiles]; };
  auto next_tile = [&](uint32_t t) {
    for (; t < total; t += gridDim.x)
      if (active(t)) return t;
    return total;
  };
  // tile geometry
  struct TG {
    uint32_t b, a;
    int64_t s0, base;
    V* buf;
    const V* src;
  };
  auto geo = [&](uint32_t t) {
    TG r;
    r.b = t / tiles;
    const uint32_t tt = t - r.b * tiles;
    r.a = tt / spt;
    r.s0 = (int64_t)(tt - r.a * spt) * lv.C;
    r.base = r.a * (int64_t)lv.F * lv.S + r.s0;
    if (DIR < 0) r.buf = X + r.b * g.NC;
    else r.buf = reinterpret_cast<V*>(imfs + r.b * g.sig_stride + (int64_t)c.M[r.b] * g.n);
    r.src = KIND == PASS_FWD_FIRST ? reinterpret_cast<const V*>(sig + r.b * g.n) : r.buf;
    return r;
  };
  // (C a power of two dividing the block: a thread's column is fixed and its digit advances by a constant,
  // so the source address advances by a constant too -- one 64-bit add per element)
  const bool fixc = lv.cs >= 0 && lv.C <= kColThreads;
  auto issue = [&](const TG& q, V* dst) {
    if constexpr (RMk) {  // F rows of C contiguous values: one bulk copy each, by the first F threads
      const int bi = (int)((dst - S[0]) / bufsz);
      const uint32_t rowb = (uint32_t)(lv.C * sizeof(V));
      if (tmode) {  // (the buffer's generic-proxy accesses were fenced by every thread before the last barrier)
        if (threadIdx.x == 0) {
          mbar_expect_tx(&cmb[bi], rowb * (uint32_t)lv.F);
          const int slot = (DIR < 0) ? (int)q.b : (int)q.b * (g.max_imfs + 1) + c.M[q.b];
          tensor_g2s(dst, &tm, (int)(q.s0 * (int64_t)(sizeof(V) / 8)), (int)(q.a * (uint32_t)lv.F), slot, &cmb[bi]);
        }
        return;
      }
      if (threadIdx.x == 0) mbar_expect_tx(&cmb[bi], rowb * (uint32_t)lv.F);
      for (int f = threadIdx.x; f < lv.F; f += blockDim.x) {
        fence_proxy_async();  // this buffer's generic-proxy reads (ordered by the last barrier) precede the copy
        bulk_g2s(dst + f * lv.C, q.src + q.base + (int64_t)f * lv.S, rowb, &cmb[bi]);
      }
      return;
    }
    if (fixc) {
      const int cc = threadIdx.x & (lv.C - 1), f0 = threadIdx.x >> lv.cs, df = kColThreads >> lv.cs;
      const V* src = q.src + q.base + (int64_t)f0 * lv.S + cc;
      const int64_t step = (int64_t)df * lv.S;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int f = f0 + j * df;
        if (f < lv.F) cp_async<(int)sizeof(V)>(dst + sidx<V>(cc, f, lv.pitch, lv.swz), src);
        src += step;
      }
      return;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = threadIdx.x + j * kColThreads;
      if (i < FC) {
        int f, cc;
        tile_fc(lv, i, f, cc);
        cp_async<(int)sizeof(V)>(dst + sidx<V>(cc, f, lv.pitch, lv.swz), q.src + q.base + (int64_t)f * lv.S + cc);
      }
    }
  };
  if constexpr (RMk) {
    if (threadIdx.x == 0) {
      mbar_init(&cmb[0], 1);
      mbar_init(&cmb[1], 1);
      mbar_init(&cmb[2], 1);
      mbar_fence_init();
    }
    __syncthreads();
  }
  uint32_t mph = 0;  // RMk: bit i = parity of the next wait on cmb[i]
  uint32_t t = next_tile(blockIdx.x);
  TG cur{};
  if (t < total) {
    cur = geo(t);
    issue(cur, S[0]);
  }
  if constexpr (!RMk) cp_async_commit();
  for (int it = 0; t < total; ++it) {
    const uint32_t tn = next_tile(t + gridDim.x);
    TG nxt{};
    if (tn < total) {
      nxt = geo(tn);
      issue(nxt, S[(it + 1) % 3]);
    }
    if constexpr (RMk) {
      const int bi = it % 3;
      mbar_wait(&cmb[bi], (mph >> bi) & 1u);
      mph ^= 1u << bi;
    } else {
      cp_async_commit();
      cp_async_wait<1>();
    }
    __syncthreads();
    V* In = S[it % 3];
    V* Sc = S[(it + 2) % 3];
    Real* Rb = imfs + cur.b * g.sig_stride + (int64_t)g.max_imfs * g.n;
    if (KIND == PASS_FWD_FIRST) {
      bool finite = true;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int i = threadIdx.x + j * kColThreads;
        if (i < FC) {
          int f, cc;
          tile_fc(lv, i, f, cc);
          const V x = In[TI(cc, f)];
          finite &= isfinite(x.x) && isfinite(x.y);
          reinterpret_cast<V*>(Rb)[cur.base + (int64_t)f * lv.S + cc] = x;
          // (row-major tiles: a column-major swizzled copy in the scratch buffer for the segment reduction)
          if (RMk) Sc[sidx<V>(cc, f, lv.pitch, lv.swz)] = x;
        }
      }
      if (!finite) atomicOr(c.bad + cur.b, 1);
      if (RMk) __syncthreads();
      const V* Sg = RMk ? Sc : In;
      if (!tile_segments_thr<Real>(Sg, lv, cur.b * g.nseg + cur.s0 / lv.C, spt, c.segi, reinterpret_cast<Real*>(c.segv)))
        tile_segments<Real>(Sg, lv, cur.b * g.nseg + cur.s0 / lv.C, spt, c.segi, reinterpret_cast<Real*>(c.segv));
    }
    V r[KIND == PASS_INV_LAST ? U : 1];
    if (KIND == PASS_INV_LAST) {  // remainder loads in flight during the transform (clamped: no local array)
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int i = threadIdx.x + j * kColThreads;
        int f, cc;
        tile_fc(lv, i < FC ? i : 0, f, cc);
        r[j] = reinterpret_cast<const V*>(Rb)[cur.base + (int64_t)f * lv.S + cc];
      }
    }
    V* out = col_fft<DIR, V, CS>(In, Sc, lvs, lv.C, tws);
    if (KIND == PASS_INV_LAST) {
      V* stage = out == In ? Sc : In;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int i = threadIdx.x + j * kColThreads;
        if (i < FC) {
          int f, cc;
          tile_fc(lv, i, f, cc);
          const int64_t gi = cur.base + (int64_t)f * lv.S + cc;
          const V x = out[TI(cc, f)];
          __stcs(cur.buf + gi, x);
          const V rn = csub(r[j], x);
          reinterpret_cast<V*>(Rb)[gi] = rn;
          // (the new remainder is staged column-major swizzled in every mode: the layout is this kernel's
          // choice here, and the thread-chunk segment reduction reads it conflict-free)
          stage[sidx<V>(cc, f, lv.pitch, lv.swz)] = rn;
        }
      }
      __syncthreads();
      if (!tile_segments_thr<Real>(stage, lv, cur.b * g.nseg + cur.s0 / lv.C, spt, c.segi, reinterpret_cast<Real*>(c.segv)))
        tile_segments<Real>(stage, lv, cur.b * g.nseg + cur.s0 / lv.C, spt, c.segi, reinterpret_cast<Real*>(c.segv));
    } else {
      // forward: this level's twiddle e^{-2 pi i s k/(F S)}; inverse: the next coarser level's
      // e^{+2 pi i s' k'/(F' S')} with s' = f S + s, k' = a mod F'.  When C divides the block size a
      // thread's column cc is fixed and its digit f advances by kColThreads/C per element, so the
      // twiddles form a geometric sequence: two table products per thread, one multiply per element.
      const int64_t kn = DIR > 0 ? (int64_t)(cur.a % (uint32_t)lvn.F) : 0;
      const bool geom = lv.cs >= 0 && lv.C <= kColThreads;
      V w{(Real)1, (Real)0}, ws{(Real)1, (Real)0};
      if (geom) {
        int f0, c0;
        tile_fc(lv, threadIdx.x, f0, c0);
        const int64_t df = kColThreads >> lv.cs;
        if (DIR < 0) {
          w = cconj(Er(tb, g.eb, lv.E2 * (cur.s0 + c0) * f0));
          ws = cconj(Er(tb, g.eb, mod2n(g, lv.E2 * ((cur.s0 + c0) * df))));
        } else {
          w = Er(tb, g.eb, mod2n(g, lvn.E2 * (((int64_t)f0 * lv.S + cur.s0 + c0) * kn)));
          ws = Er(tb, g.eb, mod2n(g, lvn.E2 * (df * lv.S * kn)));
        }
      }
      if (geom) {  // (fixc: the thread's column is fixed, its digit and address advance by constants)
        const int cc = threadIdx.x & (lv.C - 1), f0 = threadIdx.x >> lv.cs, df = kColThreads >> lv.cs;
        V* dstp = cur.buf + cur.base + (int64_t)f0 * lv.S + cc;
        const int64_t step = (int64_t)df * lv.S;
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int f = f0 + j * df;
          if (f < lv.F) {
            const V x = out[TI(cc, f)];
            *dstp = cmul(x, w);
            w = cmul(w, ws);
          }
          dstp += step;
        }
      } else
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int i = threadIdx.x + j * kColThreads;
        if (i < FC) {
          int f, cc;
          tile_fc(lv, i, f, cc);
          V x = out[TI(cc, f)];
          if (geom) {
            x = cmul(x, w);
            w = cmul(w, ws);
          } else if (DIR < 0) {
            x = cmul(x, cconj(Er(tb, g.eb, lv.E2 * (cur.s0 + cc) * f)));
          } else {
            x = cmul(x, Er(tb, g.eb, mod2n(g, lvn.E2 * (((int64_t)f * lv.S + cur.s0 + cc) * kn))));
          }
          cur.buf[cur.base + (int64_t)f * lv.S + cc] = x;
        }
      }
    }
    if constexpr (RMk) {
      if (tmode) fence_proxy_async();  // this thread's shared-memory accesses precede the tensor copies that refill
    }
    __syncthreads();
    t = tn;
    cur = nxt;
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------ a2/a3/a7 fold of extrema partials
// Groups of segments -> group partials; the last CTA of a signal folds the groups, gets k, and
// decides.  mode 0: after the forward transform (k of s); mode 1: after IMF M (bookkeeping first).
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_fold(const __grid_constant__ Geo g, const __grid_constant__ Ctl c, int mode, int32_t* __restrict__ lens,
                                                   int32_t* __restrict__ iters) {
  __shared__ Mono sm[kNW];
  __shared__ int last;
  const Real* segv = reinterpret_cast<const Real*>(c.segv);
  Real* gv = reinterpret_cast<Real*>(c.gv);
  if (blockIdx.x == 0 && threadIdx.x == 0) *c.scnt = 0;  // the next IMF's search list starts empty
  for (int64_t t = blockIdx.x; t < g.batch * g.ngrp; t += gridDim.x) {
    const int64_t b = t / g.ngrp, j = t - b * g.ngrp;
    if (!c.active[b]) continue;
    const int64_t s0 = b * g.nseg + j * g.grp, s1 = min(s0 + g.grp, (b + 1) * g.nseg);
    const Mono m = fold_items<Real>(c.segi, segv, s0, s1, sm);
    if (threadIdx.x == 0) {
      c.gi[b * g.ngrp + j] = mpack(m);
      gv[2 * (b * g.ngrp + j)] = __ldcg(segv + 2 * s0);
      gv[2 * (b * g.ngrp + j) + 1] = __ldcg(segv + 2 * (s1 - 1) + 1);
      __threadfence();
      last = atomicAdd(c.cnt + b, 1u) == (uint32_t)(g.ngrp - 1);
    }
    __syncthreads();
    if (last) {
      __threadfence();
      const Mono k = fold_items<Real>(c.gi, gv, b * g.ngrp, (b + 1) * g.ngrp, sm);
      if (threadIdx.x == 0) {
        c.cnt[b] = 0;
        int M = c.M[b];
        if (mode == 0) {
          if (c.bad[b]) {
            c.M[b] = -1;
            c.active[b] = 0;
          }
        } else {
          lens[b * g.max_imfs + M] = 2 * c.L[b];
          iters[b * g.max_imfs + M] = c.N[b];
          c.M[b] = ++M;
        }
        if (c.active[b]) {
          c.k[b] = k.c;
          if (k.c < 2 || M >= g.max_imfs) c.active[b] = 0;
          else {
            if (!g.mask) c.L[b] = filter_half_length(g, k.c);  // (mask = 1: k_peak2 sets L)
            c.search[b] = 0;
          }
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ a1 rows (forward) + post-processing
// Unit u: rows with bases u and (P - u) mod P (one row when they coincide).  After the row DFTs:
// X_k = E + e^{-2 pi i k/n} O, X_{NC-k} = conj(E - e^{-2 pi i k/n} O), E = (Z_k + conj Z_{NC-k})/2,
// O = -i (Z_k - conj Z_{NC-k})/2;  X_0 = Re Z_0 + Im Z_0, X_NC = Re Z_0 - Im Z_0 (Nyquist).
template <typename Real>
__device__ __forceinline__ void pair_of(const Geo& g, int64_t u, int64_t& ra, int64_t& rb, int64_t& bA, int& two) {
  bA = u;
  const int2 r = __ldg(g.utab + u);
  ra = r.x;
  rb = r.y;
  two = ra != rb;
}
// mirror element of t (row a) and whether the pair is processed from t
__device__ __forceinline__ bool mirror_t(const Geo& g, int64_t bA, int two, int F, int t, int& tm) {
  if (bA == 0) {
    tm = t == 0 ? 0 : F - t;
    return two || t <= tm;
  }
  tm = F - 1 - t;
  return two || t <= tm;
}

template <typename Real, int RS = 0>
__global__ void __launch_bounds__(kThreads, FIF_ST_MINB) k_rows_fwd(const __grid_constant__ Geo g, const __grid_constant__ Level lv, typename Cx<Real>::V* __restrict__ X,
                                                       typename Cx<Real>::V* __restrict__ Xn,
                                                       const __grid_constant__ Tabs<Real> tb,
                                                       const __grid_constant__ Ctl c) {
  using V = typename Cx<Real>::V;
  extern __shared__ __align__(128) char smem_raw[];
  V* A = reinterpret_cast<V*>(smem_raw);
  V* Bf = A + 2 * lv.pitch;
  const int F = lv.F;
  const uint32_t units = (uint32_t)g.units;
  for (uint32_t t = blockIdx.x; t < (uint32_t)(g.batch * g.units); t += gridDim.x) {
    const uint32_t b = t / units, u = t - b * units;
    if (!c.active[b]) continue;
    int64_t ra, rb, bA;
    int two;
    pair_of<Real>(g, u, ra, rb, bA, two);
    V* Xb = X + b * g.NC;
    {
      constexpr int UR = TileCap<Real>::value / 2 / kThreads;
      // the mirror row is loaded unconditionally (the row itself when there is none): a conditionally
      // assigned register array is kept in local memory, which serialises the loads behind its spills
      const int64_t rbb = two ? rb : ra;
      V xa[UR], xb[UR];
#pragma unroll
      for (int j = 0; j < UR; ++j) {
        const int i = threadIdx.x + j * kThreads;
        const int ic = i < F ? i : 0;
        xa[j] = Xb[ra * F + ic];
        xb[j] = Xb[rbb * F + ic];
      }
#pragma unroll
      for (int j = 0; j < UR; ++j) {
        const int i = threadIdx.x + j * kThreads;
        if (i < F) {
          A[sidx<V>(0, i, lv.pitch, lv.swz)] = xa[j];
          if (two) A[sidx<V>(1, i, lv.pitch, lv.swz)] = xb[j];
        }
      }
    }
    V* out = row_fft<-1, V, RS>(A, Bf, lv, two ? 2 : 1, tb.tw);
    V* stage = out == A ? Bf : A;
    const int cb = two ? 1 : 0;
    for (int i = threadIdx.x; i < F; i += blockDim.x) {
      int tm;
      if (!mirror_t(g, bA, two, F, i, tm)) continue;
      const int64_t k = bA + g.P * i;
      const V Pv = out[sidx<V>(0, i, lv.pitch, lv.swz)], Q = out[sidx<V>(cb, tm, lv.pitch, lv.swz)];
      if (k == 0) {
        stage[sidx<V>(0, 0, lv.pitch, lv.swz)] = V{Pv.x + Pv.y, (Real)0};
        Xn[b] = V{Pv.x - Pv.y, (Real)0};
        continue;
      }
      const Real h = (Real)0.5;
      const V E = V{h * (Pv.x + Q.x), h * (Pv.y - Q.y)};
      const V D = V{h * (Pv.x - Q.x), h * (Pv.y + Q.y)};
      const V O = V{D.y, -D.x};
      const V TO = cmul(cconj(Er(tb, g.eb, 2 * k)), O);
      stage[sidx<V>(0, i, lv.pitch, lv.swz)] = cadd(E, TO);
      stage[sidx<V>(cb, tm, lv.pitch, lv.swz)] = cconj(csub(E, TO));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < F; i += blockDim.x) {
      Xb[ra * F + i] = stage[sidx<V>(0, i, lv.pitch, lv.swz)];
      if (two) Xb[rb * F + i] = stage[sidx<V>(1, i, lv.pitch, lv.swz)];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ a6 damping + pre-processing + row IDFTs
// d = a^N (a = 1 - w_hat); X_out = (1 - d) X_in; with A = d_k X_k/n, B = d_{NC-k} X_{NC-k}/n:
// Z_k = S + T, Z_{NC-k} = conj(S - T), S = A + conj B, T = i e^{2 pi i k/n} (A - conj B)
// (k = 0 pairs with the Nyquist bin), then the length-F IDFT of each row into the IMF slot.
// SPEC = 1 (relative SD rule): the a5 cap probe is fused in -- N = cap is assumed (the common case,
// 70-97% of IMFs), the Parseval sums P, Q at the cap are accumulated from the same a^{cap-1}, and
// the last CTA of a signal decides; if SD(cap) <= delta the damping was speculative: `redo` is set,
// the K-ary search reads the untouched X_in, and a SPEC = 0 launch with redo_only recomputes X_out
// and the IMF slot for those signals.  X_in / X_out (and the Nyquist bins) ping-pong per IMF.
template <typename Real, int CAP, int SPEC, int RS = 0>
__global__ void __launch_bounds__(kThreads, FIF_ROWS_MINB) k_rows_inv(
    const __grid_constant__ Geo g, const __grid_constant__ Level lv, const __grid_constant__ Level lvn,
    Real* __restrict__ imfs,
    const typename Cx<Real>::V* __restrict__ Xin, typename Cx<Real>::V* __restrict__ Xout,
    const typename Cx<Real>::V* __restrict__ Xnin, typename Cx<Real>::V* __restrict__ Xnout,
    const __grid_constant__ Tabs<Real> tb, const __grid_constant__ Ctl c, int redo_only) {
  using V = typename Cx<Real>::V;
  extern __shared__ __align__(128) char smem_raw[];
  __shared__ double sred[kNW][2];
  __shared__ int last;
  __shared__ __align__(8) uint64_t mbar[2];
  const int F = lv.F;
  // two staging buffers for the unit's rows (filled by the bulk-copy engine, linear row layout) and the
  // FFT's first buffer; the current staging buffer doubles as the FFT's second one once it is read
  const size_t rowbuf = 2 * (size_t)lv.pitch;
  V* St0 = reinterpret_cast<V*>(smem_raw);
  V* Bf = St0 + 2 * rowbuf;
  const double invn = 1.0 / (double)g.n;
  const uint32_t units = (uint32_t)g.units;
  // redo launch: only the listed signals (SD(cap) <= delta)
  const uint32_t ntile = (!SPEC && redo_only) ? (uint32_t)(*c.scnt) * units : (uint32_t)(g.batch * g.units);
  auto sig_of = [&](uint32_t t) -> uint32_t {
    const uint32_t b = t / units;
    return (!SPEC && redo_only) ? (uint32_t)c.slist[b] : b;
  };
  auto wanted = [&](uint32_t t) {
    const uint32_t b = sig_of(t);
    return c.active[b] && !(!SPEC && redo_only && !c.redo[b]);
  };
  auto next = [&](uint32_t t) {
    for (; t < ntile; t += gridDim.x)
      if (wanted(t)) return t;
    return ntile;
  };
  // one thread issues the unit's row copies: one bulk copy per (contiguous) row, completion on mbar[stg]
  auto issue = [&](uint32_t t, int stg) {
    const uint32_t b = sig_of(t), u = t % units;
    int64_t ra, rb, bA;
    int two;
    pair_of<Real>(g, u, ra, rb, bA, two);
    const V* Xb = Xin + (int64_t)b * g.NC;
    const uint32_t rowb = (uint32_t)(F * sizeof(V));
    V* dst = St0 + stg * rowbuf;
    mbar_expect_tx(&mbar[stg], two ? 2 * rowb : rowb);
    bulk_g2s(dst, Xb + ra * F, rowb, &mbar[stg]);
    if (two) bulk_g2s(dst + F, Xb + rb * F, rowb, &mbar[stg]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  // per-thread constants of the window / twiddle recurrences (bin k = base + P i, i = tid + j blockDim)
  const double2 Ekstep = E64(tb.Eh, tb.El, g.eb, (int64_t)g.P * blockDim.x);  // e^{i pi P blockDim/n}
  uint32_t t = next(blockIdx.x);
  if (threadIdx.x == 0 && t < ntile) issue(t, 0);
  uint32_t phase = 0;  // bit s: parity of the next wait on mbar[s]
  for (int it = 0; t < ntile; ++it) {
    const int cs = it & 1;
    const uint32_t tn = next(t + gridDim.x);
    if (threadIdx.x == 0 && tn < ntile) {
      fence_proxy_async();  // the other buffer's generic-proxy use (last iteration's FFT) precedes the copy
      issue(tn, cs ^ 1);
    }
    const uint32_t b = sig_of(t), u = t % units;
    int64_t ra, rb, bA;
    int two;
    pair_of<Real>(g, u, ra, rb, bA, two);
    const int L = c.L[b], N = SPEC ? g.max_inner : c.N[b];
    V* Xo = Xout + (int64_t)b * g.NC;
    V* A = St0 + cs * rowbuf;
    const int cb = two ? 1 : 0;
    double sP = 0.0, sQ = 0.0;
    float sPf = 0.f, sQf = 0.f;  // fp32 plans: the thread's partial sums (reading A14)
    // e^{i pi k/n} and e^{i pi L k/n} advance geometrically over the thread's bins (a few complex products
    // instead of two scattered table gathers per bin pair): sin(pi k/n) = Im, sin(pi r_k/n) = |Im e^{i pi Lk/n}|
    // (the table reads are issued before the wait for the rows, so their latency overlaps the copy)
    const int64_t k0 = bA + g.P * (int64_t)threadIdx.x;
    const int64_t n2 = 2 * g.n;
    double2 Ek = E64(tb.Eh, tb.El, g.eb, k0);
    double2 Sk = E64(tb.Eh, tb.El, g.eb, mod_n((int64_t)L * k0 % n2, n2, 0.5 * invn));
    const double2 Ss = E64(tb.Eh, tb.El, g.eb, ((int64_t)L * ((g.P * blockDim.x) % n2)) % n2);
    const V xn0 = Xnin[b];
    mbar_wait(&mbar[cs], (phase >> cs) & 1u);
    phase ^= 1u << cs;
    const int P32 = (int)g.P, bA32 = (int)bA;
    for (int i = threadIdx.x; i < F; i += blockDim.x, Ek = cmul(Ek, Ekstep), Sk = cmul(Sk, Ss)) {
      int tm;
      if (!mirror_t(g, bA, two, F, i, tm)) continue;
      const int k = bA32 + P32 * i;
      const V xk = A[i];
      const V xm = k == 0 ? xn0 : A[cb * F + tm];
      double wk, wm;
      {
        const double nk = fabs(Sk.y), nm = (L & 1) ? fabs(Sk.x) : fabs(Sk.y);
        const double dk = Ek.y, dm = Ek.x;
        const double Ld = (double)L;
        double sk, sm;
        if (k == 0) {
          sk = 1.0;
          sm = nm / (Ld * dm);
        } else {
          const double inv = 1.0 / (Ld * Ld * dk * dm);
          sk = nk * Ld * dm * inv;
          sm = nm * Ld * dk * inv;
        }
        sk *= sk;
        sm *= sm;
        wk = sk * sk;
        wm = sm * sm;
      }
      Real dkr, dmr;  // a^N of the pair, rounded to Real
      V E2v;          // e^{2 pi i k/n}
      const bool self = !two && i == tm && k != 0;  // a self-paired bin (k = NC - k) is counted once
      if constexpr (sizeof(Real) == 4) {
        const float wkf = (float)wk, wmf = (float)wm;
        const float lk = log2_1m(wkf), lm = log2_1m(wmf);
        float dkf, dmf;
        if (SPEC) {
          const int m1 = (CAP > 0 ? CAP : N) - 1;
          const float ek = pow_l2(lk, m1), em = pow_l2(lm, m1);  // a^{cap-1}
          const float ck = k == 0 ? 1.f : 2.f, cm = self ? 0.f : (k == 0 ? 1.f : 2.f);
          const float pk = ck * fmaf(xk.x, xk.x, xk.y * xk.y) * (ek * ek);
          const float pm = cm * fmaf(xm.x, xm.x, xm.y * xm.y) * (em * em);
          sPf += pk + pm;
          sQf += fmaf(pk, wkf * wkf, pm * (wmf * wmf));
          dkf = ek * fmaxf(1.f - wkf, 0.f);
          dmf = em * fmaxf(1.f - wmf, 0.f);
        } else {
          dkf = pow_l2(lk, N);
          dmf = pow_l2(lm, N);
        }
        if (g.gamma > 0.0) {  // gamma-threshold (A19)
          if (dkf >= (float)(1.0 - g.gamma)) dkf = 1.f;
          if (dmf >= (float)(1.0 - g.gamma)) dmf = 1.f;
        }
        dkr = dkf;
        dmr = dmf;
        const V Ekf = V{(Real)Ek.x, (Real)Ek.y};
        E2v = cmul(Ekf, Ekf);
      } else {
      const double ak = 1.0 - wk, am = 1.0 - wm;
      double dk, dm;
      if (SPEC) {
        double ek, em;  // a^{cap-1}
        if (CAP > 0) {
          ek = upow_c<(CAP > 0 ? CAP - 1 : 1)>(ak);
          em = upow_c<(CAP > 0 ? CAP - 1 : 1)>(am);
        } else {
          ek = upow_rt(ak, N - 1);
          em = upow_rt(am, N - 1);
        }
        // Parseval weights c_k: 1 for k = 0 and the Nyquist bin, 2 otherwise
        const double ck = k == 0 ? 1.0 : 2.0, cm = self ? 0.0 : (k == 0 ? 1.0 : 2.0);
        const double pk = ck * ((double)xk.x * (double)xk.x + (double)xk.y * (double)xk.y) * (ek * ek);
        const double pm = cm * ((double)xm.x * (double)xm.x + (double)xm.y * (double)xm.y) * (em * em);
        sP += pk + pm;
        sQ += pk * wk * wk + pm * wm * wm;
        dk = ek * ak;
        dm = em * am;
      } else if (CAP > 0 && N == CAP) {
        dk = upow_c<(CAP > 0 ? CAP : 1)>(ak);
        dm = upow_c<(CAP > 0 ? CAP : 1)>(am);
      } else {
        dk = upow_rt(ak, N);
        dm = upow_rt(am, N);
      }
      if (g.gamma > 0.0) {  // gamma-threshold (A19)
        if (dk >= 1.0 - g.gamma) dk = 1.0;
        if (dm >= 1.0 - g.gamma) dm = 1.0;
      }
      dkr = (Real)dk;
      dmr = (Real)dm;
      const double2 E2k = cmul(Ek, Ek);  // e^{2 pi i k/n}
      E2v = V{(Real)E2k.x, (Real)E2k.y};
      }
      const V Av = cscale(xk, dkr * (Real)invn), Bv = cscale(xm, dmr * (Real)invn);
      const V S = V{Av.x + Bv.x, Av.y - Bv.y};
      const V D = V{Av.x - Bv.x, Av.y + Bv.y};
      const V T = mul_i<1>(cmul(E2v, D));
      Bf[sidx<V>(0, i, lv.pitch, lv.swz)] = cadd(S, T);
      Xo[ra * F + i] = cscale(xk, (Real)1 - dkr);
      if (k == 0) {
        Xnout[b] = cscale(xm, (Real)1 - dmr);
      } else {
        Bf[sidx<V>(cb, tm, lv.pitch, lv.swz)] = cconj(csub(S, T));
        Xo[(two ? rb : ra) * F + tm] = cscale(xm, (Real)1 - dmr);
      }
    }
    if (SPEC) {  // unit partial sums -> c.red, last CTA of the signal decides (fixed order)
      if constexpr (sizeof(Real) == 4) {
        sP = (double)sPf;
        sQ = (double)sQf;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sP += __shfl_xor_sync(0xffffffffu, sP, o);
        sQ += __shfl_xor_sync(0xffffffffu, sQ, o);
      }
      if ((threadIdx.x & 31) == 0) {
        sred[threadIdx.x >> 5][0] = sP;
        sred[threadIdx.x >> 5][1] = sQ;
      }
    }
    // (its first barrier publishes Bf and sred and ends every read of A, which becomes its second buffer)
    V* out = row_fft<1, V, RS>(Bf, A, lv, two ? 2 : 1, tb.tw);
    V* W = reinterpret_cast<V*>(imfs + (int64_t)b * g.sig_stride + (int64_t)c.M[b] * g.n);
    // the next (coarser) level's conjugate twiddle e^{+2 pi i s k'/(F' S')}: s = element, k' = row mod F'
    // (geometric in i: two table products per row and thread, one multiply per element)
    const int64_t ka = ra % lvn.F, kb = rb % lvn.F;
    V wa = Er(tb, g.eb, mod2n(g, lvn.E2 * ((int64_t)threadIdx.x * ka))), wb = Er(tb, g.eb, mod2n(g, lvn.E2 * ((int64_t)threadIdx.x * kb)));
    const V sa = Er(tb, g.eb, mod2n(g, lvn.E2 * ((int64_t)blockDim.x * ka)));
    const V sb = Er(tb, g.eb, mod2n(g, lvn.E2 * ((int64_t)blockDim.x * kb)));
    for (int i = threadIdx.x; i < F; i += blockDim.x) {
      W[ra * F + i] = cmul(out[sidx<V>(0, i, lv.pitch, lv.swz)], wa);
      wa = cmul(wa, sa);
      if (two) {
        W[rb * F + i] = cmul(out[sidx<V>(1, i, lv.pitch, lv.swz)], wb);
        wb = cmul(wb, sb);
      }
    }
    if (SPEC) {
      if (threadIdx.x < 2) {
        double v = 0.0;
        for (int w = 0; w < kNW; ++w) v += sred[w][threadIdx.x];
        c.red[((int64_t)b * g.nbch + u) * (2 * kProbes) + threadIdx.x] = v;
        __threadfence();  // (only the writers fence: their partials are visible before the counter moves)
      }
      __syncthreads();
      if (threadIdx.x == 0) last = atomicAdd(c.cnt + b, 1u) == (uint32_t)(g.units - 1);
      __syncthreads();
      if (last) {
        __threadfence();
        double s2[2] = {0.0, 0.0};
        const int64_t per = (g.units + blockDim.x - 1) / blockDim.x;
        const int64_t a0 = (int64_t)threadIdx.x * per, a1 = min(a0 + per, g.units);
        for (int64_t q = a0; q < a1; ++q)
#pragma unroll
          for (int i2 = 0; i2 < 2; ++i2) s2[i2] += __ldcg(c.red + ((int64_t)b * g.nbch + q) * (2 * kProbes) + i2);
        __syncthreads();
#pragma unroll
        for (int i2 = 0; i2 < 2; ++i2) {
          double v = s2[i2];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5][i2] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          double Pv = 0.0, Qv = 0.0;
          for (int w = 0; w < kNW; ++w) {
            Pv += sred[w][0];
            Qv += sred[w][1];
          }
          c.cnt[b] = 0;
          c.N[b] = g.max_inner;
          c.redo[b] = 0;
          if (Qv <= g.delta2 * Pv && g.max_inner > 1) {  // SD(cap) <= delta: search [1, cap), redo
            c.lo[b] = 0;
            c.hi[b] = g.max_inner;
            c.search[b] = 1;
            c.redo[b] = 1;
            c.slist[atomicAdd(c.scnt, 1)] = (int32_t)b;
          }
        }
      }
    }
    __syncthreads();
    t = tn;
  }
}

// ------------------------------------------------------------------ a5 probes
// mode 0: cap probe (P, Q at N = max_inner); mode 1: K-ary probes N_i = lo + i*step, i = 1..kProbes.
// One CTA per row-pair unit (both bins of every Hermitian pair share one window evaluation); the
// last CTA of a signal folds the unit partials (fixed order) and decides.
template <typename Real, int CAP, int MODE>
__global__ void __launch_bounds__(kThreads, MODE == 1 ? FIF_PROBE1_MINB : 3) k_probe(const __grid_constant__ Geo g,
                                                       const typename Cx<Real>::V* __restrict__ X,
                                                       const typename Cx<Real>::V* __restrict__ Xn,
                                                       const __grid_constant__ Tabs<Real> tb,
                                                       const __grid_constant__ Ctl c) {
  constexpr int mode = MODE;
  constexpr int NV = MODE == 0 ? 2 : 2 * kProbes;
  using V = typename Cx<Real>::V;
  __shared__ double sred[kNW][2 * kProbes];
  __shared__ int last;
  const int F = g.Frow;
  const double invn = 1.0 / (double)g.n;
  const uint32_t nbch = (uint32_t)g.nbch;
  // K-ary rounds (mode 1) visit only the listed signals
  const uint32_t ntile = MODE == 1 ? (uint32_t)(*c.scnt) * nbch : (uint32_t)(g.batch * g.nbch);
  for (uint32_t t = blockIdx.x; t < ntile; t += gridDim.x) {
    uint32_t b = t / nbch;
    const uint32_t ch = t - b * nbch;
    if (MODE == 1) b = (uint32_t)c.slist[b];
    if (!c.active[b] || (mode == 1 && !c.search[b])) continue;
    const int L = c.L[b];
    int N0, step;
    if (mode == 0) {
      N0 = g.max_inner; step = 0;
    } else {
      const int lo = c.lo[b], hi = c.hi[b];
      step = (hi - lo + kProbes) / (kProbes + 1);
      if (step < 1) step = 1;
      N0 = lo + step;
    }
    double acc[NV];
    float accf[MODE == 1 && sizeof(Real) == 4 ? NV : 1];  // fp32 plans' K-ary partial sums
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0.0;
#pragma unroll
    for (int i = 0; i < (int)(sizeof(accf) / sizeof(float)); ++i) accf[i] = 0.f;
    int64_t ra, rb, bA;
    int two;
    pair_of<Real>(g, ch, ra, rb, bA, two);
    const V* Xb = X + b * g.NC;
    constexpr int UR = TileCap<Real>::value / 2 / kThreads;
    V xkv[UR], xmv[UR];
#pragma unroll
    for (int j = 0; j < UR; ++j) {  // unconditional loads (clamped indices): the arrays stay in registers
      const int i = threadIdx.x + j * kThreads;
      const int ic = i < F ? i : 0;
      int tm;
      mirror_t(g, bA, two, F, ic, tm);
      xkv[j] = Xb[ra * F + ic];
      xmv[j] = Xb[(two ? rb : ra) * F + tm];
      if (bA == 0 && ic == 0) xmv[j] = Xn[b];
    }
    const int n32 = (int)g.n, P32 = (int)g.P, bA32 = (int)bA;  // 32-bit bin arithmetic (n <= 2^27)
    int mk = (int)mod_n((int64_t)L * (bA + g.P * threadIdx.x), g.n, invn);
    const int mstep = (int)mod_n((int64_t)L * ((g.P * kThreads) % g.n), g.n, invn);
#pragma unroll
    for (int j = 0; j < UR; ++j, mk = (mk + mstep >= n32) ? mk + mstep - n32 : mk + mstep) {
      const int i = threadIdx.x + j * kThreads;
      int tm;
      if (i >= F || !mirror_t(g, bA, two, F, i, tm)) continue;
      const int k = bA32 + P32 * i;
      const V xk = xkv[j];
      const V xm = xmv[j];
      double wk, wm;
      double2 Ek;
      what_pair_m(g, tb, L, k, mk, wk, wm, Ek);
      // Parseval weights c_k: 1 for k = 0 and the Nyquist bin, 2 otherwise; a self-paired bin
      // (k = NC - k) is counted once
      const bool self = !two && i == tm && k != 0;
      const double ck = k == 0 ? 1.0 : 2.0, cm = self ? 0.0 : (k == 0 ? 1.0 : 2.0);
      const double pk = ck * ((double)xk.x * (double)xk.x + (double)xk.y * (double)xk.y);
      const double pm = cm * ((double)xm.x * (double)xm.x + (double)xm.y * (double)xm.y);
      const double ak = 1.0 - wk, am = 1.0 - wm;
      if (MODE == 0 && g.stop == 1) {  // N0 rule: max |X_k|^2 (A16)
        acc[0] = fmax(acc[0], fmax(pk / ck, cm > 0.0 ? pm / cm : 0.0));
      } else if constexpr (MODE == 0) {
        double ek, em;
        if (CAP > 0 && N0 == CAP) {
          ek = upow_c<CAP - 1>(ak);
          em = upow_c<CAP - 1>(am);
        } else {
          ek = upow_rt(ak, N0 - 1);
          em = upow_rt(am, N0 - 1);
        }
        ek *= ek;
        em *= em;
        acc[0] += pk * ek + pm * em;
        acc[1] += pk * wk * wk * ek + pm * wm * wm * em;
      } else if constexpr (sizeof(Real) == 4) {  // fp32 plans: terms and the thread's sums in fp32 (A14)
        const float wkf = (float)wk, wmf = (float)wm;
        const float lk = log2_1m(wkf), lm = log2_1m(wmf);
        float yk = pow_l2(lk, 2 * (N0 - 1)), ym = pow_l2(lm, 2 * (N0 - 1));
        const float zk = pow_l2(lk, 2 * step), zm = pow_l2(lm, 2 * step);
        const float ck = k == 0 ? 1.f : 2.f, cm = self ? 0.f : (k == 0 ? 1.f : 2.f);
        const float pkf = ck * fmaf(xk.x, xk.x, xk.y * xk.y), pmf = cm * fmaf(xm.x, xm.x, xm.y * xm.y);
        const float qk = pkf * (wkf * wkf), qm = pmf * (wmf * wmf);
#pragma unroll
        for (int q = 0; q < kProbes; ++q) {
          accf[2 * q] += fmaf(pkf, yk, pmf * ym);
          accf[2 * q + 1] += fmaf(qk, yk, qm * ym);
          yk *= zk;
          ym *= zm;
        }
      } else {
        const double a2k = ak * ak, a2m = am * am;
        double yk = upow_rt(a2k, N0 - 1), ym = upow_rt(a2m, N0 - 1);
        const double zk = upow_rt(a2k, step), zm = upow_rt(a2m, step);
        const double qk = pk * wk * wk, qm = pm * wm * wm;
#pragma unroll
        for (int q = 0; q < kProbes; ++q) {
          acc[2 * q] += pk * yk + pm * ym;
          acc[2 * q + 1] += qk * yk + qm * ym;
          yk *= zk;
          ym *= zm;
        }
      }
    }
    if constexpr (MODE == 1 && sizeof(Real) == 4) {
#pragma unroll
      for (int i = 0; i < NV; ++i) acc[i] = (double)accf[i];
    }
    constexpr int nv = NV;
    const bool useMax = MODE == 0 && g.stop == 1;
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
    if (threadIdx.x < nv) {
      double v = 0.0;
      for (int w = 0; w < kNW; ++w) v = useMax ? fmax(v, sred[w][threadIdx.x]) : v + sred[w][threadIdx.x];
      c.red[(b * g.nbch + ch) * (2 * kProbes) + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(c.cnt + b, 1u) == (uint32_t)(g.nbch - 1);
    __syncthreads();
    if (last) {
      __threadfence();
      // fold the chunk partials: thread-contiguous ranges, then a fixed-order tree
      double s[NV];
#pragma unroll
      for (int i = 0; i < NV; ++i) s[i] = 0.0;
      const int64_t per = (g.nbch + blockDim.x - 1) / blockDim.x;
      const int64_t a0 = (int64_t)threadIdx.x * per, a1 = min(a0 + per, g.nbch);
      for (int64_t q = a0; q < a1; ++q)
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const double u = __ldcg(c.red + (b * g.nbch + q) * (2 * kProbes) + i);
          s[i] = useMax ? fmax(s[i], u) : s[i] + u;
        }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        double v = s[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double u = __shfl_xor_sync(0xffffffffu, v, o);
          v = useMax ? fmax(v, u) : v + u;
        }
        if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5][i] = v;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double PQ[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          double v = 0.0;
          for (int w = 0; w < kNW; ++w) v = useMax ? fmax(v, sred[w][i]) : v + sred[w][i];
          PQ[i] = v;
        }
        c.cnt[b] = 0;
        if (useMax) {
          // N = min(N0, cap), rhs = delta / (||U^T r||_inf sqrt(n-1)), ||U^T r||_inf = max|X| / sqrt(n)
          const double rhs = g.delta / (sqrt(PQ[0] / (double)g.n) * sqrt((double)(g.n - 1)));
          c.N[b] = n0_capped(rhs, g.max_inner);
          c.search[b] = 0;
        } else if constexpr (MODE == 0) {
          c.N[b] = g.max_inner;
          if (PQ[1] <= g.delta2 * PQ[0]) {  // SD(cap) <= delta: search [1, cap)
            c.lo[b] = 0;
            c.hi[b] = g.max_inner;
            c.search[b] = g.max_inner > 1 ? 1 : 0;
            if (g.max_inner == 1) c.N[b] = 1;
          }
        } else {
          const int lo = c.lo[b], hi = c.hi[b];
          int nlo = lo, nhi = hi;
#pragma unroll
          for (int q = 0; q < kProbes; ++q) {
            const int Nq = lo + step * (q + 1);
            if (Nq >= hi) break;
            if (PQ[2 * q + 1] <= g.delta2 * PQ[2 * q]) { nhi = Nq; break; }
            nlo = Nq;
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
    __syncthreads();
  }
}

// ------------------------------------------------------------------ a3 alternative: spectral-peak rule
// (reading A20).  k_peak1: |X_k|^2 scattered to natural bin order (one CTA per row pair)
// + the per-signal max over k >= 1; k_peak2: the largest local maximum >= 1e-4 max (neighbours are
// contiguous now), folded by the last CTA of the signal into L = rule(k = 2 f*), or the signal stops
// when there is none.
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_peak1(const __grid_constant__ Geo g,
                                                    const typename Cx<Real>::V* __restrict__ X,
                                                    const typename Cx<Real>::V* __restrict__ Xn,
                                                    const __grid_constant__ Ctl c) {
  using V = typename Cx<Real>::V;
  __shared__ double sm[kNW];
  __shared__ int last;
  const int F = g.Frow;
  const uint32_t units = (uint32_t)g.units;
  for (uint32_t t = blockIdx.x; t < (uint32_t)(g.batch * g.units); t += gridDim.x) {
    const uint32_t b = t / units, u = t - b * units;
    if (!c.active[b]) continue;
    int64_t ra, rb, bA;
    int two;
    pair_of<Real>(g, u, ra, rb, bA, two);
    const V* Xb = X + b * g.NC;
    double* pn = g.pnat + b * (g.NC + 1);
    double mx = 0.0;
    for (int i = threadIdx.x; i < F; i += blockDim.x) {
      int tm;
      if (!mirror_t(g, bA, two, F, i, tm)) continue;
      const int64_t k = bA + g.P * i;
      const V xk = Xb[ra * F + i];
      const V xm = k == 0 ? Xn[b] : Xb[(two ? rb : ra) * F + tm];
      const double pk = (double)xk.x * (double)xk.x + (double)xk.y * (double)xk.y;
      const double pm = (double)xm.x * (double)xm.x + (double)xm.y * (double)xm.y;
      pn[k] = pk;
      pn[g.NC - k] = pm;  // k = 0: the Nyquist bin NC
      if (k >= 1) mx = fmax(mx, pk);
      mx = fmax(mx, pm);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = 0.0;
      for (int w = 0; w < kNW; ++w) v = fmax(v, sm[w]);
      c.red[((int64_t)b * g.nbch + u) * (2 * kProbes)] = v;
      __threadfence();
      last = atomicAdd(c.cnt + b, 1u) == (uint32_t)(g.units - 1);
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      __threadfence();
      double v = 0.0;
      for (int64_t q = 0; q < g.units; ++q) v = fmax(v, __ldcg(c.red + ((int64_t)b * g.nbch + q) * (2 * kProbes)));
      c.pmax[b] = v;
      c.cnt[b] = 0;
    }
    __syncthreads();
  }
}

template <typename Real>
__global__ void __launch_bounds__(kThreads) k_peak2(const __grid_constant__ Geo g, const __grid_constant__ Ctl c) {
  __shared__ double sm[kNW];
  __shared__ int last;
  const uint32_t units = (uint32_t)g.units;
  const int64_t chunk = (g.NC + g.units - 1) / g.units;  // bins 1..NC in `units` chunks
  for (uint32_t t = blockIdx.x; t < (uint32_t)(g.batch * g.units); t += gridDim.x) {
    const uint32_t b = t / units, u = t - b * units;
    if (!c.active[b]) continue;
    const double* pn = g.pnat + b * (g.NC + 1);
    const double M = c.pmax[b], thr = 1e-4 * M;
    const int64_t k0 = 1 + (int64_t)u * chunk, k1 = min(k0 + chunk, g.NC + 1);
    int64_t best = 0;
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
      const double pv = pn[k];
      bool ok = M > 0.0 && pv >= thr;
      if (ok && k > 1) ok = pv > pn[k - 1];
      if (ok && k < g.NC) ok = pv >= pn[k + 1];
      if (ok) best = k;
    }
    double bv = (double)best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bv = fmax(bv, __shfl_xor_sync(0xffffffffu, bv, o));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = bv;
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = 0.0;
      for (int w = 0; w < kNW; ++w) v = fmax(v, sm[w]);
      c.red[((int64_t)b * g.nbch + u) * (2 * kProbes)] = v;
      __threadfence();
      last = atomicAdd(c.cnt + b, 1u) == (uint32_t)(g.units - 1);
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      __threadfence();
      double v = 0.0;
      for (int64_t q = 0; q < g.units; ++q) v = fmax(v, __ldcg(c.red + ((int64_t)b * g.nbch + q) * (2 * kProbes)));
      c.cnt[b] = 0;
      const int fs = (int)v;
      if (fs == 0) c.active[b] = 0;  // no significant peak: the signal stops
      else c.L[b] = filter_half_length(g, 2 * fs);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ a7 final
// trend (R lives in slot max_imfs) to slot M, zeros after; counts; zero lens/iters past M
template <typename Real>
__global__ void __launch_bounds__(kThreads) k_final(const __grid_constant__ Geo g, Real* __restrict__ imfs, const __grid_constant__ Ctl c, int32_t* count,
                                                    int32_t* lens, int32_t* iters) {
  for (int64_t t = blockIdx.x; t < g.batch; t += gridDim.x) {
    const int M = c.M[t];
    Real* base = imfs + t * g.sig_stride;
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
      if (m >= M) {
        lens[t * g.max_imfs + m] = 0;
        iters[t * g.max_imfs + m] = 0;
      }
    if (threadIdx.x == 0) count[t] = M;
    __syncthreads();
  }
}

}  // namespace st
}  // namespace fifgpu
