"""GPU parity of the cluster-resident regime (one signal per thread-block cluster of P = 2, 4, 8 CTAs, r and
r_hat on chip, four-step FFT over the cluster with TMA-landed transposes; fif_cluster.cuh) against the
direct-form oracle (oracle/direct_form.py, pinned to the time-domain oracle in tests/test_oracle_pins.py),
and against the streamed regime on the same inputs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import direct_form as df  # noqa: E402
from paper_1802_01359_b200 import fif, signals  # noqa: E402
from test_gpu_parity import TAU, assert_parity, df_batch, run_gpu  # noqa: E402

CL = fif.REGIME_CLUSTER


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_native()
    torch.cuda.set_device(0)


@pytest.mark.parametrize("n", [16384, 32768, 65536])
def test_cluster_vs_direct_form(n):
    B = 6
    s = np.stack([signals.tones_signal(n, 41, i) for i in range(B)])
    plan = fif.Plan(n, B, "f64", regime=CL)
    assert plan.launch_config()["regime"] == "cluster"
    plan.close()
    gpu = run_gpu(s, regime=CL)
    ref = df_batch(s, tau=TAU["f64"])
    for b in range(B):
        assert_parity(s[b], gpu, ref, b, b)


def test_cluster_equals_streamed():
    n, B = 65536, 8
    s = signals.make_batch("cfg2", batch=B)
    a = run_gpu(s, delta=1e-4, regime=CL)
    b = run_gpu(s, delta=1e-4, regime=fif.REGIME_STREAMED)
    np.testing.assert_array_equal(a[1], b[1])
    np.testing.assert_array_equal(a[2], b[2])
    np.testing.assert_array_equal(a[3], b[3])
    for i in range(B):
        for m in range(a[1][i] + 1):
            x, y = a[0][i, m], b[0][i, m]
            assert np.linalg.norm(x - y) <= 1e-11 * max(np.linalg.norm(x), 1e-5 * np.linalg.norm(s[i]))


@pytest.mark.parity(min_full=4 / 5, min_prefix=0)  # the 1e-300 row: rounding-level decisions
def test_cluster_degenerate_and_nonfinite():
    n = 16384
    rng = np.random.default_rng(7)
    rows = [np.zeros(n), np.full(n, 2.5), np.linspace(-1, 1, n),
            np.repeat(rng.standard_normal(n // 256), 256),            # plateaus: the exact extrema rule
            signals.tones_signal(n, 42, 0)]
    s = np.stack(rows + [signals.tones_signal(n, 42, 1)])
    s[-1, 123] = np.nan
    gpu = run_gpu(s, regime=CL)
    assert int(gpu[1][-1]) == -1 and (gpu[2][-1] == 0).all()
    ref = df.decompose_batch(s[:-1])
    for b in range(len(rows)):
        assert_parity(s[b], gpu, ref, b, b)


def test_cluster_batch_beyond_grid_and_options():
    """More signals than co-resident clusters (the persistent loop), a non-default cap, delta and max_imfs."""
    n = 32768
    plan = fif.Plan(n, 1, "f64", regime=CL)
    grid = plan.launch_config()["grid"]
    plan.close()
    B = grid // 4 * 2 + 3
    s = np.stack([signals.tones_signal(n, 43, i) for i in range(B)])
    gpu = run_gpu(s, regime=CL, delta=3e-3, max_inner=57, max_imfs=6)
    idx = [0, 1, B // 2, B - 1]
    ref = df_batch(s[idx], delta=3e-3, max_inner=57, max_imfs=6)
    for i, b in enumerate(idx):
        assert_parity(s[b], gpu, ref, b, i)


def test_cluster_plan_switches_to_streamed_for_the_spectral_rule():
    """The spectral-peak rule (A20) on an AUTO plan of a cluster length: the plan becomes a streamed
    one and decomposes as the oracle does."""
    n, B = 16384, 3
    s = np.stack([signals.tones_signal(n, 44, i) for i in range(B)])
    plan = fif.Plan(n, B, "f64")
    assert plan.launch_config()["regime"] == "cluster"
    plan.set_mask_rule(fif.MASK_SPECTRAL)
    assert plan.launch_config()["regime"] == "streamed"
    x = torch.from_numpy(s).cuda()
    out = plan.alloc_outputs()
    plan.decompose(x, *out)
    torch.cuda.synchronize()
    gpu = [t.cpu().numpy() for t in out]
    plan.close()
    ref = df.decompose_batch(s, mask=df.MASK_SPECTRAL)
    for b in range(B):
        assert_parity(s[b], gpu, ref, b, b)
