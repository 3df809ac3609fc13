// fif_iterative.cu -- the "iterative" regime: Algorithm 2 (Discrete Iterative Filtering)
// run LITERALLY on the GPU -- every inner step is the circular convolution s <- s - w (*) s (PAPER.md:392,
// :409), with the relative SD computed from the iterates.  It is the GPU counterpart of the
// iterative IF the paper compares FIF against ("roughly two days" vs "less than an hour"),
// built so that the IF-vs-FIF speedup can be measured on the same hardware ("next" #4).
// Same readings as the FIF regimes (A1-A15); the window and every convolution are evaluated in IEEE fp64
// without FMA contraction (__dmul_rn / __dadd_rn) in the oracle's order, so the iterates equal the
// time-domain oracle's bit for bit; only the SD sums are reduced in a different order.
//
// One CTA per signal (persistent over the batch); the iterate, the next iterate and the window live in
// shared memory (power-of-two-free: any even n with 3 n + 4 n/4 doubles of shared memory, n <= 8192).
#include <math.h>

#include "fif_plan.h"

namespace fifgpu {
namespace it {

constexpr int kT = 512;

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];  // fixed order: identical on all threads
  return s;
}

// interior extrema count (reading A4): strict sign changes of r[j+1] - r[j], zeros dropped, no wrap
// (one warp, ordered; the count is small work next to the iteration)
__device__ int extrema(const double* r, int64_t n, int* sh) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int64_t per = (n - 1 + 31) / 32, d0 = lane * per, d1 = min(d0 + per, n - 1);
    int f = 0, l = 0, c = 0;
    for (int64_t j = d0; j < d1; ++j) {
      const double d = r[j + 1] - r[j];
      if (d == 0.0) continue;
      const int sg = d > 0.0 ? 1 : -1;
      if (f == 0) f = sg;
      if (l != 0 && sg != l) ++c;
      l = sg;
    }
    // ordered fold over lanes
    for (int off = 1; off < 32; off <<= 1) {
      const int f2 = __shfl_down_sync(0xffffffffu, f, off), l2 = __shfl_down_sync(0xffffffffu, l, off),
                c2 = __shfl_down_sync(0xffffffffu, c, off);
      if ((lane & (2 * off - 1)) == 0 && lane + off < 32) {
        c += c2 + ((l && f2 && l != f2) ? 1 : 0);
        if (!f) f = f2;
        if (l2) l = l2;
      }
    }
    if (lane == 0) sh[0] = c;
  }
  __syncthreads();
  const int k = sh[0];
  __syncthreads();
  return k;
}

// h_j = 1 - |j|/L (|j| <= L-1), / sum (sequential, the oracle's order); w = h (*) h by the direct double sum
__device__ void make_window(int L, double* h, double* w) {
  const int hl = L - 1;
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int j = -hl; j <= hl; ++j) {
      const double v = __dadd_rn(1.0, -__ddiv_rn(fabs((double)j), (double)L));
      h[j + hl] = v;
      sum = __dadd_rn(sum, v);
    }
    for (int j = 0; j < 2 * hl + 1; ++j) h[j] = __ddiv_rn(h[j], sum);
  }
  __syncthreads();
  const int H = 2 * hl;
  for (int d = -H + (int)threadIdx.x; d <= H; d += blockDim.x) {
    double acc = 0.0;
    for (int a = -hl; a <= hl; ++a) {
      const int bb = d - a;
      if (bb < -hl || bb > hl) continue;
      acc = __dadd_rn(acc, __dmul_rn(h[a + hl], h[bb + hl]));
    }
    w[d + H] = acc;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kT) k_iterative(const double* __restrict__ sig, double* __restrict__ imfs,
                                                  int32_t* count, int32_t* lens, int32_t* iters, int64_t batch,
                                                  int64_t n, double xi, double delta, int32_t max_inner,
                                                  int32_t max_imfs, int32_t window) {
  extern __shared__ __align__(16) double smd[];
  __shared__ double red[kT / 32];
  __shared__ int ish[2];
  const int64_t Hmax = 2 * ((n - 1) / 4 - 1);  // largest window half-width (L <= (n-1)/4)
  double* c = smd;                    // current iterate, periodically extended by Hmax on both sides
  double* cn = c + n + 2 * Hmax;      // next iterate
  double* r = cn + n;                 // remainder
  double* w = r + n;                  // window (<= 2 Hmax + 1 taps)
  double* h = w + 2 * Hmax + 1;       // triangle (<= Hmax + 1 taps)
  const int64_t stride = (int64_t)(max_imfs + 1) * n;
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    const double* s = sig + b * n;
    double* out = imfs + b * stride;
    bool finite = true;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      r[i] = s[i];
      finite &= isfinite(s[i]);
    }
    if (!__syncthreads_and(finite)) {
      for (int64_t i = threadIdx.x; i < stride; i += blockDim.x) out[i] = 0.0;
      for (int m = threadIdx.x; m < max_imfs; m += blockDim.x) { lens[b * max_imfs + m] = 0; iters[b * max_imfs + m] = 0; }
      if (threadIdx.x == 0) count[b] = -1;
      __syncthreads();
      continue;
    }
    int M = 0;
    while (M < max_imfs) {
      const int k = extrema(r, n, ish);
      if (k < 2) break;
      // L = clamp(floor(fl(fl(xi n)/k)), 2, (n-1)/4)  (A1, A3, A8)
      const double u = __ddiv_rn(__dmul_rn(xi, (double)n), (double)k);
      long long q = (long long)floor(u);
      long long L = window ? 2 * q : q;
      if (L < 2) L = 2;
      if (L > (n - 1) / 4) L = (n - 1) / 4;
      make_window((int)L, h, w);
      const int64_t H = 2 * (L - 1);
      double* cc = c + Hmax;  // c[i] for i in [-Hmax, n + Hmax)
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) cc[i] = r[i];
      __syncthreads();
      int N = 0;
      for (int m = 1; m <= max_inner; ++m) {
        for (int64_t i = threadIdx.x; i < H; i += blockDim.x) {  // periodic extension by H
          cc[-1 - i] = cc[n - 1 - i];
          cc[n + i] = cc[i];
        }
        __syncthreads();
        double num = 0.0, den = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
          double v = 0.0;
          for (int64_t d = -H; d <= H; ++d) v = __dadd_rn(v, __dmul_rn(w[d + H], cc[i - d]));
          const double x = __dadd_rn(cc[i], -v);  // s_{m+1} = s_m - w (*) s_m
          cn[i] = x;
          const double dd = x - cc[i];
          num += dd * dd;
          den += cc[i] * cc[i];
        }
        num = block_sum(num, red);
        den = block_sum(den, red);
        const double sd = den > 0.0 ? sqrt(num) / sqrt(den) : 0.0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) cc[i] = cn[i];
        __syncthreads();
        N = m;
        if (sd <= delta) break;
      }
      double* imf = out + (int64_t)M * n;
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        imf[i] = cc[i];
        r[i] = r[i] - cc[i];
      }
      if (threadIdx.x == 0) { lens[b * max_imfs + M] = (int32_t)(2 * L); iters[b * max_imfs + M] = N; }
      ++M;
      __syncthreads();
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[(int64_t)M * n + i] = r[i];  // trend
    for (int64_t i = (int64_t)(M + 1) * n + threadIdx.x; i < stride; i += blockDim.x) out[i] = 0.0;
    for (int m = M + threadIdx.x; m < max_imfs; m += blockDim.x) { lens[b * max_imfs + m] = 0; iters[b * max_imfs + m] = 0; }
    if (threadIdx.x == 0) count[b] = M;
    __syncthreads();
  }
}

}  // namespace it
}  // namespace fifgpu

namespace fifhost {
size_t it_smem_bytes(int64_t n) {
  const int64_t Hmax = 2 * ((n - 1) / 4 - 1);
  return sizeof(double) * (size_t)(n + 2 * Hmax + n + n + 2 * Hmax + 1 + Hmax + 1);
}
fif_status it_setup(fif_plan_s* p) {
  if (p->dtype != FIF_F64 || p->n > 8192) return FIF_ERR_UNSUPPORTED_N;
  const size_t sm = it_smem_bytes(p->n);
  if (cudaFuncSetAttribute(fifgpu::it::k_iterative, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
    return FIF_ERR_UNSUPPORTED_N;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fifgpu::it::k_iterative, fifgpu::it::kT, sm);
  p->occ = occ > 0 ? occ : 1;
  p->block = fifgpu::it::kT;
  p->smem = sm;
  return FIF_OK;
}
void it_decompose(fif_plan_s* p, const void* sig, void* imfs, int32_t* cnt, int32_t* lens, int32_t* its, int64_t batch,
                  cudaStream_t s) {
  const int64_t cap = (int64_t)p->num_sms * p->occ;
  const int grid = (int)(batch < cap ? batch : cap);
  fifgpu::it::k_iterative<<<grid, fifgpu::it::kT, p->smem, s>>>((const double*)sig, (double*)imfs, cnt, lens, its, batch,
                                                                p->n, p->xi, p->delta, p->max_inner, p->max_imfs,
                                                                (int32_t)p->window);
}
}  // namespace fifhost
