"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (a plan over the whole
batch on one GPU), where the oracle cannot run the whole decomposition:
  * config 3 (one signal, n = 2^26, streamed regime): every decision re-derived by the oracle from the GPU's
    own remainders -- the extrema count and the filter-length rule exactly (oracle.count_extrema /
    filter_half_length), N from the SD rule evaluated by Parseval on the oracle side (numpy FFT + the
    eigenvalues of the filter row, oracle/direct_form.py), the IMF spectrum against (1 - w_hat)^N times the
    remainder spectrum at every bin, and the trend by telescoping;
  * config 4 (fp32 sweep, 1 GiB per run): the full batch decomposed, sampled signals against the direct form.
"""
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import direct_form as df  # noqa: E402
from paper_1802_01359_b200 import fif, signals  # noqa: E402
from test_gpu_parity import MARGIN_THR, TAU, assert_parity, df_batch, sample_idx  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_native()
    torch.cuda.set_device(0)


def test_cfg3_full_size_every_decision():
    _every_decision(signals.cfg3_signal(0))


def test_maximum_length_every_decision():
    """The largest n a plan accepts (2^27; include/fif.h), cfg3 recipe: the same per-decision checks on the
    first 3 IMFs (each costs the oracle side two 2^27-point numpy FFTs), telescoping on all."""
    _every_decision(signals.cfg3_signal(0, n=1 << 27), check=3)


def _every_decision(s, check=10):
    n, delta, cap = s.shape[0], 1e-3, 200
    plan = fif.Plan(n, 1, "f64", delta=delta)
    assert plan.launch_config()["regime"] == "streamed"
    x = torch.from_numpy(s[None]).cuda()
    imfs, count, lens, iters = plan.alloc_outputs()
    plan.decompose(x, imfs, count, lens, iters)
    torch.cuda.synchronize()
    M, lens, iters = int(count[0]), lens.cpu().numpy()[0], iters.cpu().numpy()[0]
    assert 1 <= M <= 10
    r = s.copy()
    snorm = np.linalg.norm(s)
    c = np.full(n // 2 + 1, 2.0)
    c[0] = c[-1] = 1.0
    for m in range(M):
        if m >= check:
            r = r - imfs[0, m].cpu().numpy()
            continue
        # r here is s minus the GPU's IMFs in the GPU's own order, i.e. the GPU's remainder bit for bit;
        # the smallest difference among 2^26 noisy samples is ~1e-10 max|s|, far above rounding
        k, em = oracle.count_extrema(r)
        assert em > 1e-14, "extremum decision at rounding level"
        L = oracle.filter_half_length(1.6, n, k)
        assert lens[m] == 2 * L, (m, lens[m], L)
        N = int(iters[m])
        R = np.fft.rfft(r)
        lam = df.eigenvalues(n, L)
        a2 = np.clip(1.0 - lam, 0.0, 1.0) ** 2
        p = c * (R.real ** 2 + R.imag ** 2)

        def sd(NN):
            e = a2 ** (NN - 1)
            return math.sqrt(float(np.dot(p * lam * lam, e)) / float(np.dot(p, e)))

        sdN = sd(N)
        assert sdN <= delta * (1 + 1e-9) or N == cap, (m, N, sdN)
        if N > 1:
            assert sd(N - 1) > delta * (1 - 1e-9), (m, N)
        imf = imfs[0, m].cpu().numpy()
        I = np.fft.rfft(imf)
        D = np.clip(1.0 - lam, 0.0, 1.0) ** N * R
        err = np.linalg.norm(I - D) / max(np.linalg.norm(D), 1e-5 * math.sqrt(n) * snorm)
        assert err <= 1e-9, (m, err)
        r = r - imf
    trend = imfs[0, M].cpu().numpy()
    assert np.abs(trend - r).max() <= 1e-10 * np.abs(s).max()
    k, _ = oracle.count_extrema(r)
    assert M == 10 or k < 2
    plan.close()


@pytest.mark.parity(min_full=0.1)  # fp32: see tests/test_gpu_parity.py::test_fp32_path
@pytest.mark.parametrize("n", [1 << 10, 1 << 14, 1 << 17, 1 << 20, 3 << 14, 5 << 14])
def test_cfg4_full_batch_sampled(n):
    """Config 4 (fp32, 1 GiB batch, the bench launch) decomposed in full; every (B/64)-th signal (64-65) vs the
    direct form on the fp32-rounded input (reading A14), spread over the host's cores."""
    B = signals.cfg4_batch(n)
    s32 = signals.make_batch("cfg4", n=n)
    plan = fif.Plan(n, B, "f32")
    if plan.launch_config()["regime"] == "resident":  # as bench.py runs it
        plan.set_eigen_table(True)
    x = torch.from_numpy(s32).cuda()
    imfs, count, lens, iters = plan.alloc_outputs()
    plan.decompose(x, imfs, count, lens, iters)
    torch.cuda.synchronize()
    idx = sample_idx(B)
    it = torch.from_numpy(idx).cuda()
    gpu = [imfs[it].cpu().numpy(), count[it].cpu().numpy(), lens[it].cpu().numpy(), iters[it].cpu().numpy()]
    cnt = count.cpu().numpy()
    assert ((cnt >= 0) & (cnt <= 10)).all()
    del x, imfs
    plan.close()
    s64 = s32[idx].astype(np.float64)
    ref = df_batch(s64, tau=TAU["f32"])
    for i in range(len(idx)):
        assert_parity(s64[i], gpu, ref, i, i, "f32")


GOLDEN3 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg3_df_2p26.npz")


def test_cfg3_vs_direct_form():
    """Config 3 end to end at its full size (one n = 2^26 signal, the single-GPU streamed plan bench.py runs)
    against the direct-form oracle's own decomposition (tests/golden/cfg3_df_2p26.npz, written by
    tests/golden/make_cfg3_golden.py from oracle/direct_form.py only; Alg. 2 :401-417):
    M and every (l_m, N_m) bit-exact where the oracle's decisions are safe (all ten are: reading A21), the
    norm of every IMF and of the trend within 1e-9 relative, and the 4223 stored samples of each within
    1e-9 of max(||IMF||, 1e-5 ||s||) (a relative-L2 error <= 1e-9 implies it)."""
    g = np.load(GOLDEN3)
    s = signals.cfg3_signal(0)
    n = s.shape[0]
    assert int(g["n"]) == n
    plan = fif.Plan(n, 1, "f64", delta=1e-3)
    x = torch.from_numpy(s[None]).cuda()
    imfs, count, lens, iters = plan.alloc_outputs()
    plan.decompose(x, imfs, count, lens, iters)
    torch.cuda.synchronize()
    M = int(g["M"])
    mg = g["margins"]
    te, tsd = MARGIN_THR["f64"]
    safe = all((np.isnan(mg[m, 0]) or mg[m, 0] >= te) and (m == M or mg[m, 1] >= tsd) for m in range(M + 1))
    assert safe, mg
    assert int(count[0]) == M
    assert lens.cpu().numpy()[0].tolist() == g["l"].tolist()
    assert iters.cpu().numpy()[0].tolist() == g["N"].tolist()
    floor = 1e-5 * float(g["snorm"])
    idx = torch.from_numpy(g["idx"]).cuda()
    for m in range(M + 1):
        row = imfs[0, m]
        nrm = float(torch.linalg.vector_norm(row))
        ref_n = float(g["norms"][m])
        assert abs(nrm - ref_n) <= 1e-9 * max(ref_n, floor), (m, nrm, ref_n)
        got = row[idx].cpu().numpy()
        assert np.abs(got - g["samples"][m]).max() <= 1e-9 * max(ref_n, floor), m
    plan.close()
