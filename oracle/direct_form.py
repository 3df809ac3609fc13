"""CPU-DF: the paper's FFT direct form (FIF), plain numpy, fp64.

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this module.
It shares no code with the CUDA path (paper_1802_01359_b200/csrc).

This is the second oracle engine.  It follows PAPER.md §4 step by step:
  * eigenvalues of W = DFT of the filter row w ("by
    means of the Fast Fourier Transform since (Lambdas) is equivalent to the
    DFT of the sequence {w_1q}") -- the row is built in the time domain exactly
    as in oracle/fif_oracle.c (h sampled, /sum, h(*)h);
  * IMF = IDFT((I-D)^N DFT(s))                       (Eq. One step_algo);
  * N: "compute (One step_algo) for subsequently bigger values of N0 and stop
    whenever SD is less or equal to delta", SD evaluated
    through Parseval as a LINEAR scan N = 1, 2, ...;
  * s = s - IMF in the time domain, re-transformed for the next IMF
    (Alg. 2).
It is pinned against the time-domain oracle (fif_oracle.c) in
tests/test_oracle_pins.py and used where the literal iteration is too slow.
Readings A1-A15 are the same as fif_oracle.c.
"""
from __future__ import annotations

import math

import numpy as np

WINDOW_TRI_SQ = 0
WINDOW_TRI_SQ_WIDE = 1
STOP_SD, STOP_N0 = 0, 1


def n0_f(N: int) -> float:
    """N^N / (N+1)^(N+1) in the stable form exp(N ln(N/(N+1))) / (N+1)."""
    return math.exp(N * math.log(N / (N + 1))) / (N + 1)


def n0_capped(rhs: float, cap: int) -> int:
    """min(N0, cap), N0 = the minimum N with n0_f(N) < rhs (Thm DIF_conv_stop)."""
    for N in range(1, cap + 1):
        if n0_f(N) < rhs:
            return N
    return cap


MASK_EXTREMA, MASK_SPECTRAL = 0, 1


def spectral_peak(rhat: np.ndarray) -> tuple:
    """(f*, margin) from the rfft bins (reading A20): the largest f in 1..n/2 that is a local
    maximum of p = |X|^2 (p_f > p_{f-1} for f > 1, p_f >= p_{f+1} for f < n/2) with p_f >= 1e-4 max p."""
    p = rhat.real ** 2 + rhat.imag ** 2
    NC = p.shape[0] - 1
    M = float(p[1:].max()) if NC >= 1 else 0.0
    thr, mg = 1e-4 * M, math.inf
    for f in range(NC, 0, -1):
        if M <= 0.0:
            break
        gap, ok = abs(p[f] - thr), p[f] >= thr
        if ok and f > 1:
            ok = p[f] > p[f - 1]
            gap = min(gap, abs(p[f] - p[f - 1]))
        if ok and f < NC:
            ok = p[f] >= p[f + 1]
            gap = min(gap, abs(p[f] - p[f + 1]))
        mg = min(mg, gap / M)
        if ok:
            return f, mg
    return 0, mg


def threshold_pin(d: np.ndarray, gamma: float) -> np.ndarray:
    """gamma-threshold: whenever (1 - w_hat)^N >= 1 - gamma, w_hat is replaced by
    zero, i.e. the damping factor becomes exactly 1 (the bin passes whole into the IMF)."""
    if gamma <= 0.0:
        return d
    return np.where(d >= 1.0 - gamma, 1.0, d)


def count_extrema(r: np.ndarray) -> int:
    """Reading A4: strict sign changes of r[j+1]-r[j], zeros dropped, no wrap."""
    d = np.diff(np.asarray(r, dtype=np.float64))
    sg = np.sign(d)
    sg = sg[sg != 0]
    return int(np.count_nonzero(sg[1:] != sg[:-1]))


def filter_half_length(xi: float, n: int, k: int, window: int = WINDOW_TRI_SQ) -> int:
    """Readings A1/A3/A8: L = clamp(floor(fl(fl(xi*n)/k)), 2, floor((n-1)/4))."""
    q = math.floor((float(xi) * float(n)) / float(k))  # Python floats are IEEE fp64, no FMA
    L = 2 * q if window == WINDOW_TRI_SQ_WIDE else q
    return int(min(max(L, 2), (n - 1) // 4))


def filter_row(n: int, L: int) -> np.ndarray:
    """Circulant row c of w = h(*)h, h_j = (1-|j|/L)/sum."""
    j = np.arange(-(L - 1), L, dtype=np.float64)
    h = 1.0 - np.abs(j) / L
    h = h / h.sum()
    w = np.convolve(h, h)  # length 4L-3, centred at index 2L-2
    H = 2 * L - 2
    row = np.zeros(n, dtype=np.float64)
    for d in range(-H, H + 1):
        row[d % n] += w[d + H]
    return row


def eigenvalues(n: int, L: int) -> np.ndarray:
    """lambda_p = DFT of the filter row (PAPER.md:543 Eq. Lambdas), real part, bins 0..n/2."""
    return np.fft.rfft(filter_row(n, L)).real


def sd_curve(rhat: np.ndarray, lam: np.ndarray, n: int, max_inner: int) -> np.ndarray:
    """SD_N for N = 1..max_inner via Parseval:
    SD_N^2 = sum c_k lam^2 a^{2(N-1)} |r_k|^2 / sum c_k a^{2(N-1)} |r_k|^2, a = 1-lam clamped to [0,1]."""
    a = np.clip(1.0 - lam, 0.0, 1.0)
    c = np.full(lam.shape, 2.0)
    c[0] = 1.0
    if n % 2 == 0:
        c[-1] = 1.0
    p = c * (rhat.real ** 2 + rhat.imag ** 2)
    q = p * lam * lam
    x = np.ones_like(a)
    a2 = a * a
    out = np.empty(max_inner)
    for N in range(1, max_inner + 1):
        P = float(np.dot(p, x))
        Q = float(np.dot(q, x))
        out[N - 1] = math.sqrt(Q) / math.sqrt(P) if P > 0.0 else 0.0
        x = x * a2
    return out


def decompose(s, xi=1.6, delta=1e-3, max_inner=200, max_imfs=10, window=WINDOW_TRI_SQ, gamma=0.0, stop=STOP_SD,
              mask=MASK_EXTREMA, tau=1e-11):
    """Full FIF decomposition of one real signal.  Returns dict with imfs [(max_imfs+1), n]
    (trend in slot M), M, l (2L per IMF), N, k (extrema counts), sd (SD_N, SD_{N-1}).
    stop = STOP_N0: N = min(N0, max_inner) from the a-priori bound with the absolute delta (PAPER.md:599,
    :611-618; readings A16-A18); gamma > 0: the threshold variant (reading A19)."""
    s = np.asarray(s, dtype=np.float64)
    n = s.shape[0]
    r = s.copy()
    imfs = np.zeros((max_imfs + 1, n))
    ls, Ns, ks, sds = [], [], [], []
    scale, snorm = float(np.abs(s).max()), float(np.linalg.norm(s))
    margins = np.full((max_imfs + 1, 2), np.nan)  # same definitions as fif_oracle.c
    M = 0
    while M < max_imfs:
        k = count_extrema(r)
        ks.append(k)
        ad = np.abs(np.diff(r))
        dd = ad[ad > 0]
        em = (dd.min() / scale) if (dd.size and scale > 0) else np.inf
        # reading A21: the first decision is on s itself; later ones are robust unless the f
        # fragile differences (|diff| <= tau max|s|, k uncertain by +-2f) could change the a3 outcome
        if M == 0:
            margins[M, 0] = np.inf
        else:
            f = int(np.count_nonzero(ad <= tau * scale))
            robust = f == 0 or (k >= 2 and k - 2 * f >= 2 and (
                mask == MASK_SPECTRAL or
                filter_half_length(xi, n, k - 2 * f, window) == filter_half_length(xi, n, k + 2 * f, window)))
            margins[M, 0] = np.inf if (robust and f > 0) else em
        if k < 2:
            break
        rhat = np.fft.rfft(r)
        if mask == MASK_SPECTRAL:  # L from k = 2 f* (A20)
            fs, pm = spectral_peak(rhat)
            margins[M, 0] = min(margins[M, 0], pm)
            if fs == 0:
                break
            L = filter_half_length(xi, n, 2 * fs, window)
        else:
            L = filter_half_length(xi, n, k, window)
        lam = eigenvalues(n, L)
        curve = sd_curve(rhat, lam, n, max_inner)
        if stop == STOP_N0:
            # ||U^T r||_inf = max_k |X_k| / sqrt(n) (unitary DFT, A16); k = 0 zero eigenvalues (A17)
            rhs = delta / (float(np.abs(rhat).max()) / math.sqrt(n) * math.sqrt(n - 1))
            N = n0_capped(rhs, max_inner)
        else:
            hit = np.nonzero(curve <= delta)[0]
            N = int(hit[0]) + 1 if hit.size else max_inner
        imf = np.fft.irfft(threshold_pin(damping(lam, N), gamma) * rhat, n)
        imfs[M] = imf
        r = r - imf
        ls.append(2 * L)
        Ns.append(N)
        sds.append((curve[N - 1], curve[N - 2] if N > 1 else float("nan")))
        # iterate norms ||(I-W)^{N-1} r|| (Parseval: sum_k c_k |a^{N-1} r_k|^2 = n ||.||^2)
        cw = np.full(lam.shape, 2.0)
        cw[0] = 1.0
        if n % 2 == 0:
            cw[-1] = 1.0
        a = np.clip(1.0 - lam, 0.0, 1.0)
        def itn(m):
            return math.sqrt(float(np.sum(cw * np.abs(a ** m * rhat) ** 2)) / n)
        if stop == STOP_N0:
            sm = abs(n0_f(N) / rhs - 1.0)
            if N > 1:
                sm = min(sm, abs(n0_f(N - 1) / rhs - 1.0))
        else:
            # reading A21: the remainder perturbation (units of ||s||) that can flip SD <= delta, first order
            sm = 0.5 * abs(curve[N - 1] - delta) * (itn(N - 1) / snorm if snorm > 0 else 1.0)
            if N > 1:
                sm = min(sm, 0.5 * abs(curve[N - 2] - delta) * (itn(N - 2) / snorm if snorm > 0 else 1.0))
        margins[M, 1] = sm
        M += 1
    if M == max_imfs:
        ks.append(count_extrema(r))
    imfs[M] = r
    return {"imfs": imfs, "M": M, "l": ls, "N": Ns, "k": ks, "sd": sds, "margins": margins}


def decompose_batch(signals, xi=1.6, delta=1e-3, max_inner=200, max_imfs=10, window=WINDOW_TRI_SQ, gamma=0.0,
                    stop=STOP_SD, mask=MASK_EXTREMA, tau=1e-11):
    """CPU-DF over a batch, returned in the TD oracle's dict layout (imfs, count, l, N, margins)."""
    S = np.atleast_2d(np.asarray(signals, dtype=np.float64))
    B, n = S.shape
    out = {"imfs": np.zeros((B, max_imfs + 1, n)), "count": np.zeros(B, np.int32),
           "l": np.zeros((B, max_imfs), np.int32), "N": np.zeros((B, max_imfs), np.int32),
           "margins": np.full((B, max_imfs + 1, 2), np.nan)}
    for b in range(B):
        d = decompose(S[b], xi, delta, max_inner, max_imfs, window, gamma, stop, mask, tau)
        M = d["M"]
        out["imfs"][b] = d["imfs"]
        out["count"][b] = M
        out["l"][b, :M] = d["l"]
        out["N"][b, :M] = d["N"]
        out["margins"][b] = d["margins"]
    return out


def damping(lam: np.ndarray, N: int) -> np.ndarray:
    """(1 - lambda)^N with 1 - lambda clamped to [0, 1] (PAPER.md:688 (I-D)^N)."""
    return np.clip(1.0 - np.asarray(lam, dtype=np.float64), 0.0, 1.0) ** N
