/*
 * oracle/fif_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, obviously-correct CPU implementation of Discrete Iterative
 * Filtering (DIF) as written in arXiv 1802.01359, in IEEE fp64.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant with the CUDA path in paper_1802_01359_b200/csrc.
 *
 * It LITERALLY ITERATES the time-domain circular convolution
 *      s_{m+1} = s_m - W s_m                       (Eq. s_m+1 / MatrixForm)
 * i.e. Algorithm 2 (DIF) with
 *   - periodic extension, W circulant
 *   - filter length fixed at the first inner step
 *   - l = 2 floor(xi * n / k)                      (Eq. Unif_Mask_length)
 *   - w = h (*) h, h triangular, rows scaled to
 *     unit sum
 *   - SD = ||s_{m+1}-s_m||_2 / ||s_m||_2 <= delta,
 *     capped at max_inner
 * No FFT is used anywhere in this file.
 *
 * Readings where the paper is silent / ambiguous:
 *   R1/A1  h has half-support L = floor(xi n / k) samples, so w = h(*)h has
 *          half-support l = 2L ("l_m ... half support length").
 *          window==1 (R3, SPEC.md:54 convention) uses L = 2 floor(xi n / k).
 *   A2     h_j = shape(j/L) = 1 - |j|/L, |j| <= L, divided by its sum.
 *   A3     L clamped to [2, floor((n-1)/4)] (PAPER.md:493 l <= (n-1)/2; lower clamp invented).
 *   A4     extrema: strict sign changes of r_{j+1}-r_j, j = 0..n-2, zero
 *          differences dropped, no wrap-around.
 *   A5     SD_N = ||(I-W)^N r - (I-W)^{N-1} r|| / ||(I-W)^{N-1} r||; stop at the
 *          first N with SD_N <= delta; IMF = (I-W)^N r (Alg. 2).
 *   A7     no N <= max_inner satisfies it -> N = max_inner.
 *   A8     floor(fl(fl(xi*n)/k)) in fp64, no contraction (compile with -ffp-contract=off).
 *   A12    trend (final remainder) stored after the M IMFs.
 *   A13    the outer loop also stops at M = max_imfs.
 *
 * Parity pins for every function: tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_WINDOW_TRI_SQ 0      /* R1 (default) */
#define ORACLE_WINDOW_TRI_SQ_WIDE 1 /* R3 */

/* ---------------------------------------------------------------------------
 * Extrema count (reading A4; PAPER.md:42 "number of extrema of s", :83 "k is the
 * number of its extreme points", SPEC.md:94 plateau rule).
 * margin_out (optional): min |Delta_j| over nonzero differences, divided by
 * `scale` (max|s| of the ORIGINAL signal; max|r| when scale <= 0) -- how far the
 * nearest sign decision is from flipping under a perturbation of relative size
 * margin (rounding differences between two correct implementations are
 * ~1e-15 max|s|, whatever the size of the remainder).
 * ------------------------------------------------------------------------- */
int64_t oracle_count_extrema(const double* r, int64_t n, double scale, double* margin_out) {
  int64_t count = 0;
  int prev = 0; /* sign of the last nonzero difference, 0 = none yet */
  double min_abs = INFINITY, max_r = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    double a = fabs(r[j]);
    if (a > max_r) max_r = a;
  }
  if (scale > 0.0) max_r = scale;
  for (int64_t j = 0; j + 1 < n; ++j) {
    double d = r[j + 1] - r[j];
    if (d == 0.0) continue; /* plateau: dropped */
    int sg = d > 0.0 ? 1 : -1;
    if (fabs(d) < min_abs) min_abs = fabs(d);
    if (prev != 0 && sg != prev) ++count;
    prev = sg;
  }
  if (margin_out) *margin_out = (max_r > 0.0 && min_abs < INFINITY) ? min_abs / max_r : INFINITY;
  return count;
}

/* ---------------------------------------------------------------------------
 * Decision margin of the a2/a3 step (reading A21): f = number of differences
 * r_{j+1} - r_j with |.| <= tau * scale (zeros included) -- those whose sign (or zero-ness) two
 * correct implementations may see differently on a remainder computed with other rounding.  Each such
 * difference changes the count by at most 2, so k' lies in [k - 2f, k + 2f].  The decision (stop when
 * k < 2, else L(k)) is ROBUST if it is the same for every k' in that range (L is monotone in k: the
 * end points decide).  Returns +INFINITY when robust, else the plain margin em.
 * ------------------------------------------------------------------------- */
int64_t oracle_filter_half_length(double xi, int64_t n, int64_t k, int window);
double oracle_extrema_decision_margin(const double* r, int64_t n, int64_t k, double em, double scale, double tau,
                                      double xi, int window, int mask_rule) {
  int64_t f = 0;
  for (int64_t j = 0; j + 1 < n; ++j)
    if (fabs(r[j + 1] - r[j]) <= tau * scale) ++f;
  if (f == 0) return em;
  if (k < 2) return em;                              /* k < 2 with fragile differences: not robust */
  const int64_t klo = k - 2 * f, khi = k + 2 * f;
  if (klo < 2) return em;                            /* the stop decision could differ */
  if (mask_rule) return INFINITY;                    /* the spectral rule only uses the stop decision */
  if (oracle_filter_half_length(xi, n, klo, window) != oracle_filter_half_length(xi, n, khi, window)) return em;
  return INFINITY;
}

/* ---------------------------------------------------------------------------
 * Filter half-length L of h (readings A1, A3, A8).  Mask length reported to the
 * user is l = 2L (PAPER.md:81 l := 2 floor(nu N / k)).
 * ------------------------------------------------------------------------- */
int64_t oracle_filter_half_length(double xi, int64_t n, int64_t k, int window) {
  volatile double t = xi * (double)n; /* fl(xi * n) */
  volatile double u = t / (double)k;  /* fl(fl(xi*n) / k) */
  int64_t q = (int64_t)floor(u);
  int64_t L = (window == ORACLE_WINDOW_TRI_SQ_WIDE) ? 2 * q : q;
  int64_t Lmax = (n - 1) / 4;
  if (L < 2) L = 2;
  if (L > Lmax) L = Lmax;
  return L;
}

/* ---------------------------------------------------------------------------
 * Window w = h (*) h (triangle PAPER.md:236-241; row scaling
 * PAPER.md:447).  h_j = 1 - |j|/L for |j| <= L (zero at |j| = L), then divided
 * by sum_j h_j.  w_d = sum_a h_a h_{d-a} by a direct double sum, |d| <= 2L-2.
 * Output: w[0 .. 2(2L-2)], w[d + (2L-2)] = w_d.  Returns the half support H=2L-2.
 * ------------------------------------------------------------------------- */
int64_t oracle_triangle(int64_t L, double* h_out /* size 2L-1 */) {
  /* h_j = shape(j/L), shape(t) = 1 - |t| (PAPER.md:236-241 with unit support), |j| <= L-1
     (h_{+-L} = 0), then divided by the sum. */
  int64_t hl = L - 1;
  double sum = 0.0;
  for (int64_t j = -hl; j <= hl; ++j) {
    double v = 1.0 - fabs((double)j) / (double)L;
    h_out[j + hl] = v;
    sum += v;
  }
  for (int64_t j = 0; j < 2 * hl + 1; ++j) h_out[j] /= sum;
  return hl;
}

int64_t oracle_window(int64_t L, double* w_out /* size 4L-3 */) {
  int64_t hl = L - 1; /* h_j nonzero for |j| <= L-1 */
  double* h = (double*)malloc(sizeof(double) * (size_t)(2 * hl + 1));
  oracle_triangle(L, h);
  int64_t H = 2 * hl;
  for (int64_t d = -H; d <= H; ++d) {
    double acc = 0.0;
    for (int64_t a = -hl; a <= hl; ++a) {
      int64_t b = d - a;
      if (b < -hl || b > hl) continue;
      acc += h[a + hl] * h[b + hl];
    }
    w_out[d + H] = acc;
  }
  free(h);
  return H;
}

/* One DIF step: out_i = c_i - sum_{|d|<=H} w_d c_{(i-d) mod n}.
 * cext is c periodically extended by H on both sides (cext[j] = c[(j-H) mod n]). */
static void dif_step(const double* cext, const double* w, int64_t H, int64_t n, double* out, int par) {
  const double* c = cext + H;
#pragma omp parallel for schedule(static) if (par)
  for (int64_t i = 0; i < n; ++i) {
    double v = 0.0;
    for (int64_t d = -H; d <= H; ++d) v += w[d + H] * c[i - d];
    out[i] = c[i] - v;
  }
}

static void extend(const double* c, int64_t n, int64_t H, double* cext) {
  /* cext[j] = c[(j - H) mod n], j = 0 .. n + 2H - 1 */
  for (int64_t j = 0; j < n + 2 * H; ++j) {
    int64_t i = (j - H) % n;
    if (i < 0) i += n;
    cext[j] = c[i];
  }
}

int64_t oracle_n0_bound(double rhs);

/* ||U^T r||_inf with U the unitary DFT matrix (reading A16: "U^T s is the DFT of s"):
 * max_k |sum_j r_j e^{-2 pi i jk/n}| / sqrt(n), by the plain O(n^2) definition (exact integer
 * reduction of jk mod n). */
double oracle_dft_inf(const double* r, int64_t n) {
  double mx = 0.0;
  const double tp = 6.283185307179586476925286766559;
  for (int64_t k = 0; k <= n / 2; ++k) {
    double re = 0.0, im = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      const int64_t m = (j * k) % n;
      const double a = tp * (double)m / (double)n;
      re += r[j] * cos(a);
      im -= r[j] * sin(a);
    }
    const double v = sqrt(re * re + im * im);
    if (v > mx) mx = v;
  }
  return mx / sqrt((double)n);
}

/* Spectral-peak filter length ("the identification of its highest frequency peak. The
 * filter length l can be chosen to be proportional to the reciprocal of this value"; reading A20):
 * p_f = |X_f|^2 (plain O(n^2) DFT), f = 1..n/2; the peak is the LARGEST f that is a local maximum
 * (p_f > p_{f-1} for f > 1, p_f >= p_{f+1} for f < n/2) with p_f >= 1e-4 max_f p_f (1% in magnitude,
 * SPEC.md:112).  Returns f* (0: no such bin -- a flat spectrum); L then follows the extrema rule with
 * k = 2 f* (a tone of f* periods has 2 f* extrema).  margin_out: the smallest relative gap
 * (/ max p) among the comparisons that decided f*. */
int64_t oracle_spectral_peak(const double* r, int64_t n, double* margin_out) {
  const int64_t NC = n / 2;
  double* p = (double*)malloc(sizeof(double) * (size_t)(NC + 2));
  const double tp = 6.283185307179586476925286766559;
  double M = 0.0;
  for (int64_t f = 1; f <= NC; ++f) {
    double re = 0.0, im = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      const int64_t m = (j * f) % n;
      const double a = tp * (double)m / (double)n;
      re += r[j] * cos(a);
      im -= r[j] * sin(a);
    }
    p[f] = re * re + im * im;
    if (p[f] > M) M = p[f];
  }
  const double thr = 1e-4 * M;
  int64_t fs = 0;
  double mg = INFINITY;
  for (int64_t f = NC; f >= 1 && M > 0.0; --f) {
    double gap = fabs(p[f] - thr);
    int ok = p[f] >= thr;
    if (ok && f > 1) { ok = p[f] > p[f - 1]; if (fabs(p[f] - p[f - 1]) < gap) gap = fabs(p[f] - p[f - 1]); }
    if (ok && f < NC) { ok = p[f] >= p[f + 1]; if (fabs(p[f] - p[f + 1]) < gap) gap = fabs(p[f] - p[f + 1]); }
    if (gap / M < mg) mg = gap / M;
    if (ok) { fs = f; break; }
  }
  if (margin_out) *margin_out = mg;
  free(p);
  return fs;
}

/* ---------------------------------------------------------------------------
 * A-priori inner loop (Thm DIF_conv_stop; the absolute criterion
 * ||s_{m+1} - s_m||_2 < delta of Eq. Discrete_Abs_StopCond): N0 = the minimum N0 with
 * N0^N0/(N0+1)^(N0+1) < delta / (||U^T r||_inf sqrt(n-1-k)), k = 0 (reading A17, SPEC.md:255's
 * conservative choice), N = min(N0, max_inner) (A18), and IMF = (I-W)^N r by N literal steps.
 * sd_out[0] = f(N0) / rhs - 1, sd_out[1] = f(N0-1) / rhs - 1 (decision margins; NaN if N0 = 1).
 * ------------------------------------------------------------------------- */
static void dif_step(const double* cext, const double* w, int64_t H, int64_t n, double* out, int par);
static void extend(const double* c, int64_t n, int64_t H, double* cext);
int32_t oracle_inner_n0(const double* r, int64_t n, int64_t L, double delta, int32_t max_inner, double* imf,
                        double* sd_out, int par) {
  const double rhs = delta / (oracle_dft_inf(r, n) * sqrt((double)(n - 1)));
  int64_t N0 = oracle_n0_bound(rhs);
  if (N0 < 0 || N0 > max_inner) N0 = max_inner;
  const int32_t N = (int32_t)N0;
  int64_t H = 2 * L - 2;
  double* w = (double*)malloc(sizeof(double) * (size_t)(2 * H + 1));
  oracle_window(L, w);
  double* cext = (double*)malloc(sizeof(double) * (size_t)(n + 2 * H));
  double* c = (double*)malloc(sizeof(double) * (size_t)n);
  double* cn = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(c, r, sizeof(double) * (size_t)n);
  for (int32_t m = 1; m <= N; ++m) {
    extend(c, n, H, cext);
    dif_step(cext, w, H, n, cn, par);
    double* t = c; c = cn; cn = t;
  }
  memcpy(imf, c, sizeof(double) * (size_t)n);
  if (sd_out) {
    const double f = exp((double)N0 * log((double)N0 / (double)(N0 + 1))) / (double)(N0 + 1);
    const double fp = N0 > 1 ? exp((double)(N0 - 1) * log((double)(N0 - 1) / (double)N0)) / (double)N0 : NAN;
    sd_out[0] = f / rhs - 1.0;
    sd_out[1] = fp / rhs - 1.0;
    sd_out[2] = sd_out[3] = 1.0;
  }
  free(w); free(cext); free(c); free(cn);
  return N;
}

/* ---------------------------------------------------------------------------
 * Inner loop (Alg. 2 inner while; SD PAPER.md:431; cap :433).
 * imf <- (I-W)^N r with N the first m in [1, max_inner] with SD_m <= delta.
 * sd_out[0] = SD_N, sd_out[1] = SD_{N-1} (NaN if N == 1), sd_out[2] = ||s_N|| (the
 * denominator of SD_N), sd_out[3] = ||s_{N-1}|| -- for margin reporting.
 * ------------------------------------------------------------------------- */
int32_t oracle_inner(const double* r, int64_t n, int64_t L, double delta, int32_t max_inner, double* imf,
                     double* sd_out, int par) {
  int64_t H = 2 * L - 2;
  double* w = (double*)malloc(sizeof(double) * (size_t)(2 * H + 1));
  oracle_window(L, w);
  double* cext = (double*)malloc(sizeof(double) * (size_t)(n + 2 * H));
  double* c = (double*)malloc(sizeof(double) * (size_t)n);
  double* cn = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(c, r, sizeof(double) * (size_t)n);
  int32_t N = 0;
  double sd = NAN, sd_prev = NAN, nrm = NAN, nrm_prev = NAN;
  for (int32_t m = 1; m <= max_inner; ++m) {
    extend(c, n, H, cext);
    dif_step(cext, w, H, n, cn, par);
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double d = cn[i] - c[i];
      num += d * d;
      den += c[i] * c[i];
    }
    sd_prev = sd;
    nrm_prev = nrm;
    sd = (den > 0.0) ? sqrt(num) / sqrt(den) : 0.0;
    nrm = sqrt(den);
    double* t = c; c = cn; cn = t; /* c <- s_{m+1} */
    N = m;
    if (sd <= delta) break;
  }
  memcpy(imf, c, sizeof(double) * (size_t)n);
  if (sd_out) { sd_out[0] = sd; sd_out[1] = sd_prev; sd_out[2] = nrm; sd_out[3] = nrm_prev; }
  free(w); free(cext); free(c); free(cn);
  return N;
}

/* ---------------------------------------------------------------------------
 * Outer loop (Alg. 2).  One signal.
 *   imfs   : [(max_imfs+1) * n]  IMF_0..IMF_{M-1}, trend in slot M, zeros after
 *   l_out  : [max_imfs]  mask length l_m = 2L (0 past M)
 *   N_out  : [max_imfs]  iteration counts (0 past M)
 *   k_out  : [max_imfs+1] extrema count at the head of outer step m (k_out[M] = final)
 *   margins: [(max_imfs+1) * 2]  per outer step m <= M: (margin of the extrema count at the
 *            head of step m, SD margin of IMF m); NaN where no such decision was taken
 * Returns M.
 * ------------------------------------------------------------------------- */
int32_t oracle_decompose_one(const double* s, int64_t n, int window, double xi, double delta, int32_t max_inner,
                             int32_t max_imfs, double* imfs, int32_t* l_out, int32_t* N_out, int32_t* k_out,
                             double* margins, int par, int stop, int mask_rule, double tau) {
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(r, s, sizeof(double) * (size_t)n);
  memset(imfs, 0, sizeof(double) * (size_t)n * (size_t)(max_imfs + 1));
  double scale = 0.0, snorm = 0.0;
  for (int64_t i = 0; i < n; ++i) { if (fabs(s[i]) > scale) scale = fabs(s[i]); snorm += s[i] * s[i]; }
  snorm = sqrt(snorm);
  for (int32_t m = 0; m < max_imfs; ++m) { l_out[m] = 0; N_out[m] = 0; }
  if (margins) for (int32_t m = 0; m <= max_imfs; ++m) { margins[2 * m] = NAN; margins[2 * m + 1] = NAN; }
  if (k_out) for (int32_t m = 0; m <= max_imfs; ++m) k_out[m] = -1;
  int32_t M = 0;
  while (M < max_imfs) {
    double em;
    int64_t k = oracle_count_extrema(r, n, scale, &em);
    if (k_out) k_out[M] = (int32_t)k;
    /* reading A21: the first count is taken on s itself (the same IEEE differences on any implementation);
       later ones on remainders, robust unless fragile differences could change the a3 outcome */
    if (margins) margins[2 * M] = (M == 0) ? INFINITY
                                           : oracle_extrema_decision_margin(r, n, k, em, scale, tau, xi, window,
                                                                            mask_rule);
    if (k < 2) break; /* trend: fewer than 2 extrema */
    int64_t L;
    if (mask_rule) {  /* spectral-peak rule (A20): L from k = 2 f* */
      double pm;
      const int64_t fs = oracle_spectral_peak(r, n, &pm);
      if (margins && pm < margins[2 * M]) margins[2 * M] = pm;
      if (fs == 0) break;
      L = oracle_filter_half_length(xi, n, 2 * fs, window);
    } else {
      L = oracle_filter_half_length(xi, n, k, window);
    }
    double sd[4];
    double* imf = imfs + (size_t)M * (size_t)n;
    int32_t N = stop ? oracle_inner_n0(r, n, L, delta, max_inner, imf, sd, par)
                     : oracle_inner(r, n, L, delta, max_inner, imf, sd, par);
    for (int64_t i = 0; i < n; ++i) r[i] -= imf[i]; /* s = s - s_m */
    l_out[M] = (int32_t)(2 * L);
    N_out[M] = N;
    if (margins && stop) {
      /* N0 rule: relative distance of f(N0), f(N0-1) to the right-hand side */
      double sm = fabs(sd[0]);
      if (!isnan(sd[1]) && fabs(sd[1]) < sm) sm = fabs(sd[1]);
      margins[2 * M + 1] = sm;
    } else if (margins) {
      /* reading A21: the remainder perturbation, in units of ||s||, that can flip the decision SD <= delta
         (to first order |dSD| <= 2 ||dr|| / ||iterate||): |SD - delta| ||iterate|| / (2 ||s||), the smaller
         of the tests at N and N - 1.  Two implementations' remainders differ by ~1e-16 ||s||, so a decision
         on a remainder at rounding level has no margin. */
      double sm = 0.5 * fabs(sd[0] - delta) * (snorm > 0.0 ? sd[2] / snorm : 1.0);
      if (!isnan(sd[1])) {
        double s1 = 0.5 * fabs(sd[1] - delta) * (snorm > 0.0 ? sd[3] / snorm : 1.0);
        if (s1 < sm) sm = s1;
      }
      margins[2 * M + 1] = sm;
    }
    ++M;
  }
  if (k_out && M == max_imfs) k_out[M] = (int32_t)oracle_count_extrema(r, n, scale, NULL);
  memcpy(imfs + (size_t)M * (size_t)n, r, sizeof(double) * (size_t)n); /* trend */
  free(r);
  return M;
}

/* Batch of independent signals [batch][n] (OpenMP across signals; within the
 * stencil when batch == 1).  Non-finite input -> count = -1, outputs zeroed. */
void oracle_decompose_batch(const double* s, int64_t batch, int64_t n, int window, double xi, double delta,
                            int32_t max_inner, int32_t max_imfs, double* imfs, int32_t* counts, int32_t* l_out,
                            int32_t* N_out, int32_t* k_out, double* margins, int stop, int mask_rule, double tau) {
  int par_inner = (batch == 1);
#pragma omp parallel for schedule(dynamic, 1) if (batch > 1)
  for (int64_t b = 0; b < batch; ++b) {
    const double* sb = s + (size_t)b * (size_t)n;
    int finite = 1;
    for (int64_t i = 0; i < n; ++i) if (!isfinite(sb[i])) { finite = 0; break; }
    double* ib = imfs + (size_t)b * (size_t)n * (size_t)(max_imfs + 1);
    int32_t* lb = l_out + (size_t)b * (size_t)max_imfs;
    int32_t* nb = N_out + (size_t)b * (size_t)max_imfs;
    int32_t* kb = k_out ? k_out + (size_t)b * (size_t)(max_imfs + 1) : NULL;
    double* mb = margins ? margins + (size_t)b * (size_t)(max_imfs + 1) * 2 : NULL;
    if (!finite) {
      memset(ib, 0, sizeof(double) * (size_t)n * (size_t)(max_imfs + 1));
      memset(lb, 0, sizeof(int32_t) * (size_t)max_imfs);
      memset(nb, 0, sizeof(int32_t) * (size_t)max_imfs);
      counts[b] = -1;
      continue;
    }
    counts[b] = oracle_decompose_one(sb, n, window, xi, delta, max_inner, max_imfs, ib, lb, nb, kb, mb, par_inner,
                                     stop, mask_rule, tau);
  }
}

/* A-priori iteration bound (Thm DIF_conv_stop, Eq. N0_discrete):
 * the minimum N0 in N with N0^N0 / (N0+1)^(N0+1) < rhs, where
 * rhs = delta / (||U^T s||_inf sqrt(n-1-k)).  Evaluated as the paper writes the
 * sequence, in the stable form exp(N0 ln(N0/(N0+1))) / (N0+1).  Returns -1 if
 * N0 would exceed 10^9. */
int64_t oracle_n0_bound(double rhs) {
  for (int64_t N0 = 1; N0 <= 1000000000LL; ++N0) {
    double f = exp((double)N0 * log((double)N0 / (double)(N0 + 1))) / (double)(N0 + 1);
    if (f < rhs) return N0;
  }
  return -1;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
