"""Pins for the oracle (oracle/fif_oracle.c, oracle/direct_form.py) against what
PAPER.md and mathematics fix -- never against the oracle itself or the CUDA path.

Each test names the passage it follows.  A plausible mistake in the oracle (a
dropped term, a wrong sign or index, a transposed operand, an off-by-one in N)
fails at least one of these:
  * window / eigenvalues: three independent routes (cosine sum PAPER.md:488,
    DFT of the row PAPER.md:543, Fejer^4 closed form) + continuous limit :245
  * dense brute force: W = Wh^2 as an explicit matrix, (I-W)^N s by
    N mat-vecs and the SD rule on n <= 64
  * pure tones: eigenvectors of W -> closed-form IMF and N
  * zero-eigenvalue tone passes unchanged
  * telescoping, no fake oscillations
  * SPEC worked examples (tests/golden/spec_examples.json)
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import direct_form as df
from paper_1802_01359_b200 import signals

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ----------------------------------------------------------------------------- helpers (independent routes)
def extrema_by_definition(x):
    """Independent definition: collapse runs of equal values, then count interior
    points of the collapsed sequence that are strict local maxima or minima."""
    c = [x[0]]
    for v in x[1:]:
        if v != c[-1]:
            c.append(v)
    k = 0
    for i in range(1, len(c) - 1):
        if (c[i] > c[i - 1] and c[i] > c[i + 1]) or (c[i] < c[i - 1] and c[i] < c[i + 1]):
            k += 1
    return k


def circ_row_from_centered(v, n):
    H = (len(v) - 1) // 2
    row = np.zeros(n)
    for d in range(-H, H + 1):
        row[d % n] += v[d + H]
    return row


def dense_circulant(row):
    """W_ij = c_{(i-j) mod n}."""
    n = len(row)
    i = np.arange(n)
    return row[(i[:, None] - i[None, :]) % n]


def fejer4(n, L, k):
    """Closed form of the DFT of w = h(*)h with h_j = (L-|j|)/L^2:
    w_hat_k = [sin(pi L k / n) / (L sin(pi k / n))]^4, w_hat_0 = 1 (derived)."""
    k = np.asarray(k)
    out = np.ones(k.shape)
    nz = (k % n) != 0
    kk = k[nz].astype(np.float64)
    m = (L * k[nz]) % n
    out[nz] = (np.sin(np.pi * m / n) / (L * np.sin(np.pi * kk / n))) ** 4
    return out


def cosine_sum_eigs(row):
    """lambda_j = c_0 + 2 sum_{k>=1} c_k cos(2 pi j k / n) (Eq. eig2; symmetric row)."""
    n = len(row)
    out = np.empty(n // 2 + 1)
    for j in range(n // 2 + 1):
        acc = row[0]
        for k in range(1, (n + 1) // 2):
            acc += 2.0 * row[k] * math.cos(2.0 * math.pi * j * k / n)
        if n % 2 == 0:
            acc += row[n // 2] * math.cos(math.pi * j)
        out[j] = acc
    return out


# ----------------------------------------------------------------------------- SPEC worked examples
@pytest.mark.parametrize("ex", GOLDEN["count_extrema"], ids=lambda e: e["cite"])
def test_count_extrema_spec_examples(ex):
    assert oracle.count_extrema(np.array(ex["signal"], float))[0] == ex["k"]
    assert df.count_extrema(np.array(ex["signal"], float)) == ex["k"]


@pytest.mark.parametrize("ex", GOLDEN["mask_length"], ids=lambda e: e["cite"])
def test_mask_length_spec_examples(ex):
    assert 2 * oracle.filter_half_length(ex["nu"], ex["n"], ex["k"]) == ex["l"]
    assert 2 * df.filter_half_length(ex["nu"], ex["n"], ex["k"]) == ex["l"]


def test_triangle_spec_example():
    ex = GOLDEN["triangle"][0]
    h = oracle.triangle(ex["L"])
    np.testing.assert_allclose(circ_row_from_centered(h, ex["n"]), ex["row"], rtol=0, atol=1e-16)


def test_n0_bound_spec_examples():
    for ex in GOLDEN["n0_bound"]:
        assert oracle.n0_bound(ex["rhs"]) == ex["N0"], ex["cite"]
    # the sequence N^N/(N+1)^(N+1) is the max of (1-l)^N l over [0,1]: check by brute force
    for N in (1, 5, 37):
        lam = np.linspace(0, 1, 200001)
        assert abs(((1 - lam) ** N * lam).max() - N ** N / (N + 1) ** (N + 1)) < 1e-9


def test_damping_spec_example():
    ex = GOLDEN["damping"][0]
    assert abs(df.damping(np.array([ex["lam"]]), ex["N"])[0] - ex["factor"]) < 1e-15


# ----------------------------------------------------------------------------- extrema / mask length
def test_count_extrema_brute_force():
    rng = np.random.default_rng(7)
    for trial in range(400):
        n = int(rng.integers(3, 40))
        x = rng.integers(-3, 4, n).astype(float)  # many ties / plateaus
        assert oracle.count_extrema(x)[0] == extrema_by_definition(list(x)), x
        assert df.count_extrema(x) == extrema_by_definition(list(x))
    for trial in range(50):
        x = rng.standard_normal(int(rng.integers(3, 500)))
        assert oracle.count_extrema(x)[0] == extrema_by_definition(list(x))


def test_filter_half_length_rule():
    """l = 2 floor(nu n / k), L clamped to [2, floor((n-1)/4)] (reading A3)."""
    rng = np.random.default_rng(3)
    checked = 0
    for _ in range(3000):
        n = int(rng.integers(9, 1 << 20))
        k = int(rng.integers(1, n))
        xi = float(rng.choice([1.6, 1.0, 2.0, 0.75, rng.uniform(0.5, 3.0)]))
        exact = Fraction(xi) * n / k
        if abs(exact - round(exact)) < Fraction(1, 10 ** 9):
            continue  # fp64 rounding may legitimately decide these (reading A8)
        q = math.floor(exact)
        L = min(max(q, 2), (n - 1) // 4)
        assert oracle.filter_half_length(xi, n, k) == L
        Lw = min(max(2 * q, 2), (n - 1) // 4)
        assert oracle.filter_half_length(xi, n, k, oracle.WINDOW_TRI_SQ_WIDE) == Lw
        checked += 1
    assert checked > 2500
    # exact-integer quotient decided in fp64 (A8): 1.6 * 81920 / 1024 = 128 exactly
    assert oracle.filter_half_length(1.6, 5 << 14, 1024) == 128


# ----------------------------------------------------------------------------- window & spectrum (P3, P4)
@pytest.mark.parametrize("L", [1, 2, 3, 5, 8, 16, 33])
def test_window_shape(L):
    """w = h(*)h: nonneg, symmetric, unit sum (Def. window); h(*)h by numpy.convolve."""
    h = oracle.triangle(L)
    w = oracle.window(L)
    assert len(w) == 4 * L - 3
    np.testing.assert_allclose(h.sum(), 1.0, atol=1e-15)
    np.testing.assert_allclose(w, np.convolve(h, h), atol=1e-17)
    np.testing.assert_allclose(w, w[::-1], atol=0)
    assert (w >= 0).all() and abs(w.sum() - 1) < 1e-14
    # h_j = (L - |j|) / L^2 (triangle of PAPER.md:238 sampled at j, unit sum)
    j = np.arange(-(L - 1), L)
    np.testing.assert_allclose(h, (L - np.abs(j)) / L ** 2, rtol=1e-14)


@pytest.mark.parametrize("n,L", [(64, 2), (65, 7), (100, 24), (257, 32), (1024, 12), (1024, 16), (4096, 1023),
                                 (3 << 10, 100), (5 << 10, 77)])
def test_eigenvalue_routes_agree(n, L):
    """Three routes: cosine sum, DFT of the row (numpy FFT) and the
    Fejer^4 closed form must agree; Thm Spectra / Cor. double convolution invariants."""
    row = circ_row_from_centered(oracle.window(L), n)
    ev_fft = np.fft.rfft(row)
    assert np.abs(ev_fft.imag).max() < 1e-14  # real spectrum
    ev_cos = cosine_sum_eigs(row) if n <= 1024 else None
    ev_cf = fejer4(n, L, np.arange(n // 2 + 1))
    np.testing.assert_allclose(ev_fft.real, ev_cf, rtol=0, atol=5e-15)
    if ev_cos is not None:
        np.testing.assert_allclose(ev_cos, ev_cf, rtol=0, atol=5e-14)
    np.testing.assert_allclose(df.eigenvalues(n, L), ev_cf, atol=5e-15)
    assert abs(ev_cf[0] - 1) < 1e-15
    assert (ev_fft.real[1:] < 1 - 1e-12).all()  # unique unit eigenvalue
    assert (ev_fft.real > -1e-15).all()         # spectrum in [0,1)


def test_delta_filter_all_ones():
    """c0 = 1 -> all eigenvalues equal 1.  L = 1 gives h = w = delta."""
    assert np.allclose(oracle.window(1), [1.0])
    assert np.allclose(df.eigenvalues(33, 1), 1.0)


def test_continuous_triangle_limit():
    """Continuous FT of the unit-area triangle of half-width a (PAPER.md:245 with L=a):
    w_hat(xi) = (1/a) sin^2(a pi xi)/(pi xi)^2 = sinc^2(a xi).  Our h at L samples on a grid of
    n points is that triangle with a = L/n, so h_hat_k -> sinc^2(L k / n) for k << n, and
    w_hat = h_hat^2."""
    n, L = 1 << 16, 512
    row = circ_row_from_centered(oracle.window(L), n)
    ev = np.fft.rfft(row).real
    k = np.arange(1, 400)
    cont = np.sinc(L * k / n) ** 4
    assert np.abs(ev[1:400] - cont).max() < 5e-5  # O((k/n)^2) + O(1/L^2) discretisation


# ----------------------------------------------------------------------------- dense brute force (P2)
@pytest.mark.parametrize("n", [16, 33, 64])
def test_dense_brute_force_inner(n):
    """(I-W)^N s with W = Wh^2 built as explicit matrices."""
    rng = np.random.default_rng(n)
    for L in range(2, (n - 1) // 4 + 1):
        Wh = dense_circulant(circ_row_from_centered(oracle.triangle(L), n))
        Wh = Wh / Wh.sum(axis=1, keepdims=True)  # scale each row by its sum
        W = Wh @ Wh
        s = rng.standard_normal(n)
        A = np.eye(n) - W
        for N in (1, 5, 50, 200):
            ref = s.copy()
            for _ in range(N):
                ref = A @ ref
            got, Ngot, _, _ = oracle.inner(s, L, 0.0, N)  # delta = 0: never stops early -> N applications
            assert Ngot == N
            assert np.abs(got - ref).max() <= 1e-12 * np.linalg.norm(s)


@pytest.mark.parametrize("n", [16, 33, 64])
def test_dense_brute_force_sd_rule(n):
    """N = first m with ||s_{m+1}-s_m|| / ||s_m|| <= delta (reading A5)."""
    rng = np.random.default_rng(100 + n)
    for L in range(2, (n - 1) // 4 + 1):
        Wh = dense_circulant(circ_row_from_centered(oracle.triangle(L), n))
        W = Wh @ Wh
        s = rng.standard_normal(n)
        for delta in (0.3, 0.1, 1e-2, 1e-3):
            c = s.copy()
            Nref = 60
            for m in range(1, 61):
                cn = c - W @ c
                sd = np.linalg.norm(cn - c) / np.linalg.norm(c)
                c = cn
                if sd <= delta:
                    Nref = m
                    break
            imf, N, sdN, _ = oracle.inner(s, L, delta, 60)
            assert N == Nref, (L, delta)
            assert np.abs(imf - c).max() <= 1e-12 * np.linalg.norm(s)


# ----------------------------------------------------------------------------- pure tones (P5, P8)
def test_zero_eigenvalue_tone_passes_unchanged():
    """w_hat_k = 0 exactly when L k = 0 mod n (n=1024, L=16, k=64): (I-W) fixes the tone, SD = 0,
    N = 1 and IMF = tone (PAPER.md:102 chi_{w_hat=0}, :559-562 Z has ones there)."""
    n, L, f = 1024, 16, 64
    x = np.cos(2 * np.pi * f * np.arange(n) / n + 0.7)
    imf, N, sd, _ = oracle.inner(x, L, 1e-3, 200)
    assert N == 1 and sd < 1e-13
    assert np.abs(imf - x).max() < 1e-13


@pytest.mark.parametrize("f,L", [(64, 12), (40, 30), (100, 7), (511, 9)])  # w_hat_f small: (1-w)^200 stays far above rounding
def test_pure_tone_closed_form(f, L):
    """A tone at bin f is an eigenvector of W: (I-W)^N x = (1-w_hat_f)^N x and
    SD_N = w_hat_f for every N, so N = 1 if w_hat_f <= delta else max_inner."""
    n = 1024
    x = np.cos(2 * np.pi * f * np.arange(n) / n + 0.3)
    wf = fejer4(n, L, np.array([f]))[0]
    for delta in (1e-3, 0.5):
        imf, N, sd, _ = oracle.inner(x, L, delta, 200)
        Nexp = 1 if wf <= delta else 200
        assert N == Nexp
        assert abs(sd - wf) <= 1e-12 + 1e-9 * wf
        np.testing.assert_allclose(imf, (1 - wf) ** N * x, atol=1e-12)


def test_pure_tone_full_pipeline():
    """n=1024, f=64, phi=0.3 through the whole outer loop: k = 127 interior extrema, L = floor(1.6*1024/127) = 12,
    IMF_1 = (1 - w_hat_64)^200 x (w_hat from the closed form)."""
    n, f = 1024, 64
    x = np.cos(2 * np.pi * f * np.arange(n) / n + 0.3)
    o = oracle.decompose(x)
    k = extrema_by_definition(list(x))
    assert o["k"][0, 0] == k
    L = math.floor(Fraction(1.6) * n / k)
    assert o["l"][0, 0] == 2 * L
    wf = fejer4(n, L, np.array([f]))[0]
    assert o["N"][0, 0] == 200
    np.testing.assert_allclose(o["imfs"][0, 0], (1 - wf) ** 200 * x, atol=1e-12)


# ----------------------------------------------------------------------------- outer loop invariants (P1, P6)
def _remainders(imfs, s, M):
    r = [s.copy()]
    for m in range(M):
        r.append(r[-1] - imfs[m])
    return r


@pytest.mark.parametrize("seed", [0, 1])
def test_telescoping_and_no_fake_oscillations(seed):
    """sum IMFs + trend = s and |DFT(IMF)_k| <= |DFT(r)_k|."""
    s = signals.cfg0_signal(seed)
    o = oracle.decompose(s)
    M = int(o["count"][0])
    imfs = o["imfs"][0]
    assert np.abs(imfs[: M + 1].sum(0) - s).max() <= 1e-13 * np.linalg.norm(s)
    assert np.all(imfs[M + 1:] == 0)
    rs = _remainders(imfs, s, M)
    for m in range(M):
        R = np.abs(np.fft.rfft(rs[m]))
        F = np.abs(np.fft.rfft(imfs[m]))
        assert (F <= R + 1e-9 * np.linalg.norm(rs[m])).all()


def test_trend_and_termination():
    """Monotone / constant signals: zero IMFs, trend = s.
    White noise terminates within max_imfs (Thm IF_outer_conv analog)."""
    n = 256
    for s in (np.linspace(-1, 2, n), np.full(n, 3.0), np.linspace(0, 1, n) ** 2):
        o = oracle.decompose(s)
        assert o["count"][0] == 0
        np.testing.assert_array_equal(o["imfs"][0, 0], s)
    noise = np.random.default_rng(5).standard_normal(4096)
    o = oracle.decompose(noise, max_imfs=10)
    assert 1 <= o["count"][0] <= 10


def test_nonfinite_input_flagged():
    s = signals.cfg0_signal(0)
    s[17] = np.nan
    o = oracle.decompose(s)
    assert o["count"][0] == -1


# ----------------------------------------------------------------------------- SD monotonicity (P7)
def test_sd_monotone_in_N():
    """SD_N^2 = E_N[w_hat^2] under weights c p a^{2(N-1)}: non-increasing in N (P7).
    This is what makes the GPU's cap-first probe + bisection equal to the paper's linear scan."""
    rng = np.random.default_rng(11)
    for _ in range(200):
        n = int(rng.choice([64, 256, 1024, 4096]))
        L = int(rng.integers(2, (n - 1) // 4 + 1))
        lam = df.eigenvalues(n, L)
        rhat = (rng.standard_normal(n // 2 + 1) + 1j * rng.standard_normal(n // 2 + 1)) * np.exp(
            rng.uniform(-8, 3, n // 2 + 1))
        curve = df.sd_curve(rhat, lam, n, 200)
        assert (np.diff(curve) <= 1e-12 * curve[:-1]).all()


# ----------------------------------------------------------------------------- the two engines agree
def test_td_vs_direct_form_cfg0():
    """The literal iteration (fif_oracle.c) and the paper's FFT direct form (direct_form.py) give
    identical integers and IMFs to ~1e-11 (the direct form is the same iterate)."""
    for s in (signals.cfg0_signal(0), signals.cfg0_signal(0, noise=0.0)):
        o = oracle.decompose(s)
        d = df.decompose(s)
        M = int(o["count"][0])
        assert M == d["M"]
        assert list(o["l"][0, :M]) == d["l"]
        assert list(o["N"][0, :M]) == d["N"]
        floor = 1e-5 * np.linalg.norm(s)
        for m in range(M + 1):
            a, b = o["imfs"][0, m], d["imfs"][m]
            assert np.linalg.norm(a - b) / max(np.linalg.norm(a), floor) < 1e-10


@pytest.mark.slow
def test_td_vs_direct_form_cfg1_sample():
    s = signals.make_batch("cfg1", batch=4)
    o = oracle.decompose(s)
    for b in range(4):
        d = df.decompose(s[b])
        M = int(o["count"][b])
        assert M == d["M"]
        assert list(o["l"][b, :M]) == d["l"] and list(o["N"][b, :M]) == d["N"]
        floor = 1e-5 * np.linalg.norm(s[b])
        for m in range(M + 1):
            a, c = o["imfs"][b, m], d["imfs"][m]
            assert np.linalg.norm(a - c) / max(np.linalg.norm(a), floor) < 1e-10


def test_wide_window_two_tone_separation():
    """SPEC acceptance #8 under reading R3 (FIF_WINDOW_TRI_SQ_WIDE): sin(2pi 4t)+sin(2pi 32t),
    n = 512: exactly two IMFs with max-abs > 0.5, correlated > 0.95 with the 32- and the 4-tone."""
    n = 512
    t = np.arange(n) / n
    hi, lo = np.sin(2 * np.pi * 32 * t), np.sin(2 * np.pi * 4 * t)
    o = oracle.decompose(hi + lo, window=oracle.WINDOW_TRI_SQ_WIDE)
    M = int(o["count"][0])
    sig = [o["imfs"][0, m] for m in range(M) if np.abs(o["imfs"][0, m]).max() > 0.5]
    assert len(sig) == 2
    assert np.corrcoef(sig[0], hi)[0, 1] > 0.95
    assert np.corrcoef(sig[1], lo)[0, 1] > 0.95


# ------------------------------------------------------------------ NEXT rows: a-priori N0 rule, gamma threshold
def test_dft_inf_is_the_unitary_dft_max():
    """oracle_dft_inf (O(n^2) definition) = max |FFT| / sqrt(n) (reading A16: U^T s is the DFT)."""
    rng = np.random.default_rng(7)
    for n in (16, 33, 100, 256):
        r = rng.standard_normal(n)
        assert abs(oracle.dft_inf(r) - np.abs(np.fft.fft(r)).max() / math.sqrt(n)) <= 1e-12 * math.sqrt(n)


def test_n0_rule_pure_tone_closed_form():
    """Pure tone A cos(2 pi f j/n + phi): ||U^T s||_inf = A sqrt(n)/2 in closed form, so N0 is fixed by
    Eq. N0_discrete without any DFT, and the IMF is (1 - w_f)^N s (tone = eigenvector)."""
    n, f, A, phi = 1024, 20, 1.7, 0.4
    x = A * np.cos(2 * np.pi * f * np.arange(n) / n + phi)
    for delta in (0.5, 2.0, 8.0):
        rhs = delta / (A * math.sqrt(n) / 2 * math.sqrt(n - 1))
        N_expect = next((N for N in range(1, 201) if N ** N / (N + 1) ** (N + 1) < rhs), 200)
        k = oracle.count_extrema(x)[0]
        L = oracle.filter_half_length(1.6, n, k)
        imf, N = oracle.inner_n0(x, L, delta, 200)
        assert N == N_expect, (delta, N, N_expect)
        wf = df.eigenvalues(n, L)[f]
        np.testing.assert_allclose(imf, (1 - wf) ** N * x, atol=1e-12)


def test_n0_rule_bound_is_sound():
    """Thm DIF_conv_stop: after N0 steps, ||s_{N0+1} - s_N0||_2 < delta (N0 below the cap)."""
    for i in range(4):
        s = signals.tones_signal(512, 41, i)
        k = oracle.count_extrema(s)[0]
        L = oracle.filter_half_length(1.6, 512, k)
        for delta in (1.0, 3.0):
            imf, N = oracle.inner_n0(s, L, delta, 10 ** 6)
            nxt = oracle.inner_n0(imf, L, 1e300, 1)[0]  # one more literal step (N0 = 1 for a huge delta)
            assert np.linalg.norm(nxt - imf) < delta, (i, delta, N)


def test_n0_rule_td_equals_direct_form():
    s = np.stack([signals.tones_signal(1024, 40, i) for i in range(3)])
    for delta in (2.0, 5.0):
        a = oracle.decompose(s, delta=delta, stop=oracle.STOP_N0)
        b = df.decompose_batch(s, delta=delta, stop=df.STOP_N0)
        np.testing.assert_array_equal(a["count"], b["count"])
        np.testing.assert_array_equal(a["l"], b["l"])
        np.testing.assert_array_equal(a["N"], b["N"])
        assert np.abs(a["imfs"] - b["imfs"]).max() <= 1e-11


def test_gamma_threshold_equivalence_spec_example():
    """gamma = 0.75, N = 2 -> threshold 1 - 0.5 = 0.5; (1-w)^N >= 1-gamma <=> w <= 1-(1-gamma)^(1/N)."""
    lam = np.linspace(0.0, 1.0, 100001)
    pinned = df.threshold_pin(df.damping(lam, 2), 0.75) == 1.0
    np.testing.assert_array_equal(pinned, lam <= 0.5)
    for gamma, N in ((0.1, 50), (0.3, 7), (0.9, 200)):
        th = 1.0 - (1.0 - gamma) ** (1.0 / N)
        pinned = df.threshold_pin(df.damping(lam, N), gamma) == 1.0
        off = np.abs(lam - th) > 1e-12
        np.testing.assert_array_equal(pinned[off], (lam <= th)[off])


def test_gamma_threshold_masked_bins_pass_whole():
    """SPEC.md:251 / PAPER.md:262 (Eq. IMF_cont_stop_threshold): bins in I_gamma pass into the IMF exactly,
    the others are damped by (1 - w)^N; the IMF is never larger than the remainder (no fake oscillations)."""
    n = 2048
    s = signals.tones_signal(n, 42, 0)
    plain = df.decompose(s, max_imfs=1)
    th = df.decompose(s, max_imfs=1, gamma=0.3)
    assert th["l"] == plain["l"] and th["N"] == plain["N"]
    L, N = th["l"][0] // 2, th["N"][0]
    lam = df.eigenvalues(n, L)
    d = np.clip(1 - lam, 0, 1) ** N
    mask = d >= 0.7
    assert mask.any() and (~mask).any()
    S, I = np.fft.rfft(s), np.fft.rfft(th["imfs"][0])
    np.testing.assert_allclose(I[mask], S[mask], atol=1e-10 * np.abs(S).max())
    np.testing.assert_allclose(I[~mask], d[~mask] * S[~mask], atol=1e-10 * np.abs(S).max())
    assert (np.abs(I) <= np.abs(S) + 1e-9 * np.abs(S).max()).all()


def test_gamma_to_zero_is_the_plain_method():
    s = signals.tones_signal(1024, 43, 0)
    a = df.decompose(s)
    b = df.decompose(s, gamma=1e-300)
    assert a["N"] == b["N"] and a["l"] == b["l"]
    assert np.abs(a["imfs"] - b["imfs"]).max() == 0.0


# ------------------------------------------------------------------ NEXT row: spectral-peak filter length
def test_spectral_peak_spec_examples():
    """a tone of 8 periods (n=256) -> peak bin 8 -> l = 32 at nu = 1; tones at bins 4 and 32
    of equal amplitude -> bin 32 -> l = 8; a constant has no peak (flat spectrum).  Our l = 2L with L from
    the extrema rule at k = 2 f* (reading A20) reproduces SPEC's l on both."""
    n = 256
    x = np.arange(n) / n
    tone = np.sin(2 * np.pi * 8 * x + 0.3)
    two = np.sin(2 * np.pi * 4 * x) + np.sin(2 * np.pi * 32 * x)
    for s, f_expect, l_expect in ((tone, 8, 32), (two, 32, 8)):
        f, _ = oracle.spectral_peak(s)
        assert f == f_expect
        assert 2 * oracle.filter_half_length(1.0, n, 2 * f) == l_expect
        assert df.spectral_peak(np.fft.rfft(s))[0] == f_expect
    # no AC content at all -> no peak (a constant never reaches the rule: it has no extrema)
    assert oracle.spectral_peak(np.zeros(n))[0] == 0


def test_spectral_peak_definition_brute_force():
    """The O(n^2) oracle = an independent numpy scan of the definition (rfft powers), random spectra."""
    rng = np.random.default_rng(11)
    for t in range(60):
        n = int(rng.choice([64, 96, 128, 250]))
        s = rng.standard_normal(n) * rng.uniform(0, 1, n) ** 3 + np.sin(2 * np.pi * rng.integers(1, n // 2) * np.arange(n) / n)
        p = np.abs(np.fft.rfft(s)) ** 2
        NC = n // 2
        thr = 1e-4 * p[1:].max()
        peaks = [f for f in range(1, NC + 1) if p[f] >= thr and (f == 1 or p[f] > p[f - 1]) and (f == NC or p[f] >= p[f + 1])]
        f, margin = oracle.spectral_peak(s)
        if margin > 1e-9:
            assert f == (max(peaks) if peaks else 0)


def test_spectral_rule_td_equals_direct_form():
    s = np.stack([signals.tones_signal(1024, 61, i, sigma=0.001) for i in range(3)])
    a = oracle.decompose(s, mask=oracle.MASK_SPECTRAL)
    b = df.decompose_batch(s, mask=df.MASK_SPECTRAL)
    np.testing.assert_array_equal(a["count"], b["count"])
    np.testing.assert_array_equal(a["l"], b["l"])
    np.testing.assert_array_equal(a["N"], b["N"])
    assert np.abs(a["imfs"] - b["imfs"]).max() <= 1e-11
    # l follows each signal's highest tone: 2 floor(xi n / (2 f*)) at the first IMF
    for b in range(3):
        f, _ = oracle.spectral_peak(s[b])
        assert a["l"][b][0] == 2 * oracle.filter_half_length(1.6, 1024, 2 * f)


# ----------------------------------------------------------------------------- decision margins (reading A21)
# The margins decide which IMFs the GPU parity tests compare (tests/test_gpu_parity.py::safe_prefix), so
# they are pinned here against hand-built cases and closed forms, and across the two oracle engines.

def test_extrema_margin_hand_built_plateaus():
    """min |nonzero diff| / max|r| on a hand-built row with plateaus (SPEC.md:94 zeros dropped):
    diffs 1, 0, -0.5, 0, 1.5, -6, -0.25 -> signs + - + - -  -> k = 3; margin 0.25 / 4.25."""
    r = np.array([0.0, 1.0, 1.0, 0.5, 0.5, 2.0, -4.0, -4.25])
    k, m = oracle.count_extrema(r)
    assert k == 3
    assert m == 0.25 / 4.25


def _zigzag_then_ramp(n, K, fragile_at=None, eps=1e-13):
    """K interior extrema (0,1,0,1,... over the first K+2 points), then a strictly increasing ramp; optionally
    one ramp step of size eps (a 'fragile' difference) or 0 (a plateau)."""
    x = np.empty(n)
    x[: K + 2] = [(j % 2) * 1.0 for j in range(K + 2)]
    base = x[K + 1]
    steps = np.full(n - K - 2, 1.0)
    if fragile_at is not None:
        steps[fragile_at] = eps
    x[K + 2:] = base + 2.0 + np.cumsum(steps)
    return x


@pytest.mark.parametrize("K,robust", [(300, True), (320, False), (100, False)])
@pytest.mark.parametrize("eps", [1e-13, 0.0])
def test_extrema_decision_margin_robustness(K, robust, eps):
    """Reading A21: f fragile differences leave k uncertain by +-2f; the decision is robust iff
    floor(fl(xi n)/k') is the same at k' = k - 2f and k + 2f (exact rational floors):
    n = 1000, xi = 1.6: 1600/298 = 5.37, 1600/302 = 5.30 (robust); 1600/318 = 5.03, 1600/322 = 4.97 (not);
    1600/98 = 16.3, 1600/102 = 15.7 (not).  Here f = 1 (one ramp step of size eps: tiny or a plateau)."""
    n = 1000
    x = _zigzag_then_ramp(n, K, fragile_at=200, eps=eps)
    k, em = oracle.count_extrema(x)
    assert k == K
    lo, hi = Fraction(1600, K - 2), Fraction(1600, K + 2)
    assert (math.floor(lo) == math.floor(hi)) == robust  # the case is what its name says
    m = oracle.extrema_decision_margin(x, k, em, np.abs(x).max(), 1e-9)
    assert (m == math.inf) == robust
    if not robust:
        assert m == em
    # no fragile difference: the plain margin whatever k
    y = _zigzag_then_ramp(n, K)
    ky, emy = oracle.count_extrema(y)
    assert oracle.extrema_decision_margin(y, ky, emy, np.abs(y).max(), 1e-9) == emy


def test_extrema_decision_margin_stop_decision():
    """k < 2 with a fragile difference, or k - 2f < 2: the stop decision is not robust."""
    x = np.arange(50.0)
    x[20] = x[19]  # one plateau step: k = 0, f = 1
    k, em = oracle.count_extrema(x)
    assert k == 0
    assert oracle.extrema_decision_margin(x, k, em, 49.0, 1e-9) == em
    y = _zigzag_then_ramp(60, 2, fragile_at=10)  # k = 2, f = 1 -> k - 2 = 0 < 2
    ky, emy = oracle.count_extrema(y)
    assert ky == 2 and oracle.extrema_decision_margin(y, ky, emy, np.abs(y).max(), 1e-9) == emy


def _fejer4(n, L, f):
    """w_hat_f in closed form (independent of the oracle): [sin(pi L f/n) / (L sin(pi f/n))]^4."""
    return (math.sin(math.pi * L * f / n) / (L * math.sin(math.pi * f / n))) ** 4


@pytest.mark.parametrize("f,delta,expect_N", [(64, 1e-3, 200), (300, 0.9, 1)])
def test_sd_margin_pure_tone_closed_form(f, delta, expect_N):
    """A pure tone is an eigenvector: SD_N = w_hat_f for every N, the iterate norms are
    (1 - w_hat)^(N-1) ||s||, so the SD margin (reading A21: |SD - delta| ||iterate|| / (2 ||s||), the
    smaller of the decisions at N and N - 1) is |w - delta| (1 - w)^(N-1) / 2 with N = cap = 200 when
    w > delta, and |w - delta| / 2 at N = 1 when w <= delta.  The first extrema decision is on s: +inf."""
    n = 1024
    s = np.cos(2 * np.pi * f * np.arange(n) / n + 0.3)
    r = oracle.decompose(s, delta=delta, max_imfs=1)
    k = int(r["k"][0, 0])
    L = oracle.filter_half_length(1.6, n, k)
    w = _fejer4(n, L, f)
    assert int(r["N"][0, 0]) == expect_N
    want = 0.5 * abs(w - delta) * ((1 - w) ** (expect_N - 1) if expect_N > 1 else 1.0)
    assert r["margins"][0, 0, 0] == math.inf
    assert r["margins"][0, 0, 1] == pytest.approx(want, rel=1e-9)


def test_margins_td_equal_direct_form():
    """The two oracle engines report the same margins (definitions of reading A21 evaluated once by the literal
    iteration, once through Parseval): cfg0 (noisy and noise-free) and 3 cfg1 signals; margins above the
    rounding level agree to 1e-6 relative, +inf where one is +inf."""
    rows = [signals.make_batch("cfg0")[0], signals.cfg0_signal(0, noise=0.0)] + list(signals.make_batch("cfg1", batch=3))
    for s in rows:
        td = oracle.decompose(s)
        dfr = df.decompose(s)
        M = int(td["count"][0])
        assert M == dfr["M"]
        a, b = td["margins"][0][: M + 1], dfr["margins"][: M + 1]
        for m in range(M + 1):
            for c in range(2):
                x, y = a[m, c], b[m, c]
                if np.isnan(x) or np.isnan(y):
                    assert np.isnan(x) and np.isnan(y)
                elif math.isinf(x) or math.isinf(y):
                    assert x == y
                elif max(x, y) > 1e-9:
                    assert x == pytest.approx(y, rel=1e-6), (m, c, x, y)


# ----------------------------------------------------------------------------- noise-free cfg0 fixture
SURVEY_E9 = {  # SURVEY.md §8c "Noise-free cfg0 fixture (R1 readings, TD literal; E9)": an independent
    "k": [128, 128, 128, 112, 32, 32, 20, 4, 4, 4],  # throwaway numpy model written during the survey
    "l": [24, 24, 24, 28, 102, 102, 162, 510, 510, 510],
    "N": [200, 200, 200, 8, 200, 200, 200, 50, 150, 200],
    "M": 10,
}


def test_noise_free_cfg0_golden_matches_survey_and_oracle():
    """tests/golden/cfg0_noise_free.json (written by make_cfg0_golden.py from oracle/ only) equals the survey's
    independent computation, and the oracle as it stands still reproduces it (Alg. 2,
    PAPER.md:401-417)."""
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg0_noise_free.json")))
    assert g["M"] == SURVEY_E9["M"]
    assert g["k"][: g["M"]] == SURVEY_E9["k"]
    assert g["l"] == SURVEY_E9["l"] and g["N"] == SURVEY_E9["N"]
    s = signals.cfg0_signal(0, noise=0.0)
    r = oracle.decompose(s)
    assert int(r["count"][0]) == g["M"]
    assert r["l"][0].tolist() == g["l"] and r["N"][0].tolist() == g["N"]
