"""GPU parity of the method options (SURVEY.md §8f "next" rows) in every regime:
  * the a-priori N0 stopping rule (Thm DIF_conv_stop; absolute delta, readings A16-A18)
    against the literal time-domain oracle (which iterates exactly N = min(N0, max_inner) times);
  * the gamma-threshold variant (reading A19) against the paper's direct form
    (oracle/direct_form.py; the threshold is a spectral operation, so the literal oracle has none).
Same protocol as test_gpu_parity.py (integers exact, IMFs <= 1e-9 fp64 / 2e-4 fp32, margin screening)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import direct_form as df  # noqa: E402
from paper_1802_01359_b200 import fif, signals  # noqa: E402
from test_gpu_parity import TAU, assert_parity  # noqa: E402
from test_gpu_dist import run_dist  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_native()
    torch.cuda.set_device(0)


def run_opt(s, stop=0, gamma=0.0, dtype="f64", regime=fif.REGIME_AUTO, **kw):
    s = np.ascontiguousarray(s)
    plan = fif.Plan(s.shape[1], s.shape[0], dtype, regime=regime, **kw).set_options(stop, gamma)
    x = torch.from_numpy(s).cuda()
    out = plan.alloc_outputs()
    plan.decompose(x, *out)
    torch.cuda.synchronize()
    res = [t.cpu().numpy() for t in out]
    plan.close()
    return res


REGIMES = [("resident", fif.REGIME_RESIDENT, 4096), ("streamed", fif.REGIME_STREAMED, 4096),
           ("streamed-3x", fif.REGIME_STREAMED, 3 * 1024)]


@pytest.mark.parametrize("name,regime,n", REGIMES)
@pytest.mark.parametrize("delta", [8.0, 20.0])
def test_n0_rule_vs_td_oracle(name, regime, n, delta):
    s = np.stack([signals.tones_signal(n, 50, i) for i in range(4)])
    gpu = run_opt(s, stop=fif.STOP_N0, regime=regime, delta=delta)
    ref = oracle.decompose(s, delta=delta, stop=oracle.STOP_N0)
    assert (ref["N"][:, :3] < 200).all()  # the rule, not the cap, decides
    for b in range(4):
        assert_parity(s[b], gpu, ref, b, b)


@pytest.mark.parametrize("name,regime,n", REGIMES)
@pytest.mark.parametrize("gamma", [0.1, 0.4])
def test_gamma_threshold_vs_direct_form(name, regime, n, gamma):
    s = np.stack([signals.tones_signal(n, 51, i) for i in range(4)])
    gpu = run_opt(s, gamma=gamma, regime=regime)
    ref = df.decompose_batch(s, gamma=gamma)
    for b in range(4):
        assert_parity(s[b], gpu, ref, b, b)


@pytest.mark.parity(min_full=0.1)  # fp32: see tests/test_gpu_parity.py::test_fp32_path
def test_gamma_and_n0_combined_fp32():
    n = 1 << 14
    s32 = np.stack([signals.cfg4_signal(n, i) for i in range(3)])
    gpu = run_opt(s32, stop=fif.STOP_N0, gamma=0.2, dtype="f32", delta=20.0)
    s64 = s32.astype(np.float64)
    ref = df.decompose_batch(s64, delta=20.0, gamma=0.2, stop=df.STOP_N0, tau=TAU["f32"])
    for b in range(3):
        assert_parity(s64[b], gpu, ref, b, b, "f32")


@pytest.mark.parametrize("P", [2, 4])
def test_options_distributed(P):
    n = 4096
    s = signals.tones_signal(n, 52, 0)
    plan = fif.Plan.dist(n, 0, P, emulated=True, delta=20.0).set_options(fif.STOP_N0, 0.25)
    x = torch.from_numpy(np.ascontiguousarray(s.reshape(P, n // P))).cuda()
    imfs, count, lens, iters = plan.alloc_outputs()
    plan.decompose(x, imfs, count, lens, iters)
    torch.cuda.synchronize()
    full = np.concatenate(list(imfs.cpu().numpy()), axis=1)[None]
    gpu = [full, count.cpu().numpy()[:1], lens.cpu().numpy()[:1], iters.cpu().numpy()[:1]]
    plan.close()
    ref = df.decompose_batch(s[None], delta=20.0, gamma=0.25, stop=df.STOP_N0)
    assert_parity(s, gpu, ref, 0, 0)


def test_options_validation():
    plan = fif.Plan(1024, 1)
    for stop, gamma in ((2, 0.0), (0, -0.1), (0, 1.0), (0, float("nan"))):
        with pytest.raises(fif.FifError):
            plan.set_options(stop, gamma)
    plan.close()


@pytest.mark.parametrize("name,regime,n", REGIMES)
def test_spectral_peak_rule_vs_td_oracle(name, regime, n):
    """Filter length from the highest significant spectral peak (reading A20)."""
    s = np.stack([signals.tones_signal(n, 53, i, sigma=0.001) for i in range(4)])
    s[3] = signals.tones_signal(n, 53, 3)  # sigma = 0.05: noise bins above 1% -> small L, many IMFs
    plan = fif.Plan(n, 4, "f64", regime=regime).set_mask_rule(fif.MASK_SPECTRAL)
    x = torch.from_numpy(s).cuda()
    out = plan.alloc_outputs()
    plan.decompose(x, *out)
    torch.cuda.synchronize()
    gpu = [t.cpu().numpy() for t in out]
    plan.close()
    ref = oracle.decompose(s, mask=oracle.MASK_SPECTRAL)
    for b in range(4):
        assert_parity(s[b], gpu, ref, b, b)


@pytest.mark.parity(min_full=0.1)  # fp32: see tests/test_gpu_parity.py::test_fp32_path
def test_spectral_peak_rule_fp32_and_dist_unsupported():
    n = 1 << 14
    s32 = np.stack([signals.cfg4_signal(n, i) for i in range(2)])
    plan = fif.Plan(n, 2, "f32").set_mask_rule(fif.MASK_SPECTRAL)
    x = torch.from_numpy(s32).cuda()
    out = plan.alloc_outputs()
    plan.decompose(x, *out)
    torch.cuda.synchronize()
    gpu = [t.cpu().numpy() for t in out]
    plan.close()
    s64 = s32.astype(np.float64)
    ref = df.decompose_batch(s64, mask=df.MASK_SPECTRAL, tau=TAU["f32"])
    for b in range(2):
        assert_parity(s64[b], gpu, ref, b, b, "f32")
    dp = fif.Plan.dist(4096, 0, 2, emulated=True)
    with pytest.raises(fif.FifError):
        dp.set_mask_rule(fif.MASK_SPECTRAL)
    dp.close()


# ------------------------------------------------------------------ per-L eigenvalue table
@pytest.mark.parametrize("n,dtype", [(1024, "f64"), (4096, "f64"), (8192, "f64"), (4096, "f32"), (16384, "f32")])
def test_eigen_table_bit_identical(n, dtype):
    """eigenvalues precomputed for every scaling L; the table is filled by the kernel's own
    window code, so the decomposition must not change by a single bit (64 signals: many distinct L)."""
    B = 64
    s = np.stack([signals.tones_signal(n, 41, i) for i in range(B)])
    td = torch.float64 if dtype == "f64" else torch.float32
    x = torch.from_numpy(s).to(td).cuda()
    outs = []
    for eig in (False, True):
        plan = fif.Plan(n, B, dtype)
        assert plan.launch_config()["regime"] == "resident"
        if eig:
            plan.set_eigen_table(True)
        out = plan.alloc_outputs()
        plan.decompose(x, *out)
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy() for t in out])
        plan.close()
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)
    assert len(set(outs[0][2].ravel().tolist())) > 8  # many filter lengths exercised


def test_eigen_table_with_options_and_toggle():
    n, B = 4096, 32
    s = signals.make_batch("cfg1", batch=B, start=700)
    x = torch.from_numpy(s).cuda()
    for stop, gamma, mask in ((fif.STOP_N0, 0.0, fif.MASK_EXTREMA), (fif.STOP_SD, 0.05, fif.MASK_EXTREMA),
                              (fif.STOP_SD, 0.0, fif.MASK_SPECTRAL)):
        res = []
        for eig in (False, True, False):
            plan = fif.Plan(n, B, "f64", delta=20.0 if stop == fif.STOP_N0 else 1e-3)
            plan.set_options(stop=stop, gamma=gamma).set_mask_rule(mask)
            if eig:
                plan.set_eigen_table(True)
            out = plan.alloc_outputs()
            plan.decompose(x, *out)
            if eig:  # toggled off again: back to the closed form
                plan.set_eigen_table(False)
                out2 = plan.alloc_outputs()
                plan.decompose(x, *out2)
                torch.cuda.synchronize()
                for a, b in zip(out, out2):
                    assert torch.equal(a, b)
            torch.cuda.synchronize()
            res.append([t.cpu().numpy() for t in out])
            plan.close()
        for a, b in zip(res[0], res[1]):
            np.testing.assert_array_equal(a, b)


def test_eigen_table_regimes():
    st = fif.Plan(16384, 2, "f64", regime=fif.REGIME_STREAMED)
    assert fif.lib().fif_plan_set_eigen_table(st.handle, 1) == 2
    assert fif.lib().fif_plan_set_eigen_table(st.handle, 0) == 0
