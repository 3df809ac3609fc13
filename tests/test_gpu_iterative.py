"""GPU parity of the iterative regime: Algorithm 2 run literally on the GPU -- the IF
baseline the paper measures FIF against.  Its window and convolutions follow the
time-domain oracle operation for operation (fp64, no FMA contraction), so the iterates agree to rounding
of the SD reductions only; integers bit-exact (margin-screened as everywhere)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_1802_01359_b200 import fif, signals  # noqa: E402
from test_gpu_parity import assert_parity, run_gpu  # noqa: E402

IT = fif.REGIME_ITERATIVE


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_native()
    torch.cuda.set_device(0)


def test_iterative_cfg0_vs_td_oracle():
    s = signals.make_batch("cfg0")
    gpu = run_gpu(s, regime=IT)
    ref = oracle.decompose(s)
    assert_parity(s[0], gpu, ref, 0, 0)
    M = int(ref["count"][0])
    assert np.abs(gpu[0][0, : M + 1] - ref["imfs"][0, : M + 1]).max() <= 1e-12 * np.abs(s).max()


@pytest.mark.parametrize("n", [512, 2048, 3 * 1024])
def test_iterative_vs_td_oracle(n):
    s = np.stack([signals.tones_signal(n, 70, i) for i in range(3)])
    gpu = run_gpu(s, regime=IT, max_imfs=4)
    ref = oracle.decompose(s, max_imfs=4)
    for b in range(3):
        assert_parity(s[b], gpu, ref, b, b)


def test_iterative_equals_fif_integers():
    """Same method, two algorithms (literal iteration vs the FFT direct form): identical decisions."""
    s = signals.make_batch("cfg1", batch=8, start=40)
    a = run_gpu(s, regime=IT, max_imfs=3)
    b = run_gpu(s, regime=fif.REGIME_RESIDENT, max_imfs=3)
    np.testing.assert_array_equal(a[1], b[1])
    np.testing.assert_array_equal(a[2], b[2])
    np.testing.assert_array_equal(a[3], b[3])
    for i in range(8):
        for m in range(a[1][i] + 1):
            x, y = a[0][i, m], b[0][i, m]
            assert np.linalg.norm(x - y) <= 1e-9 * max(np.linalg.norm(x), 1e-5 * np.linalg.norm(s[i]))


def test_iterative_degenerate_and_options():
    n = 1024
    rows = [np.zeros(n), np.full(n, 2.0), np.linspace(0, 1, n), signals.tones_signal(n, 71, 0)]
    s = np.stack(rows)
    s[3, 5] = np.nan
    imfs, count, _, _ = run_gpu(s, regime=IT)
    assert count[3] == -1 and (imfs[3] == 0).all()
    ref = oracle.decompose(s[:3])
    for b in range(3):
        assert count[b] == ref["count"][b] == 0
        np.testing.assert_array_equal(imfs[b, 0], s[b])
    plan = fif.Plan(n, 1, regime=IT)
    with pytest.raises(fif.FifError):
        plan.set_options(fif.STOP_N0, 0.0)
    with pytest.raises(fif.FifError):
        plan.set_mask_rule(fif.MASK_SPECTRAL)
    plan.close()
    with pytest.raises(fif.FifError):
        fif.Plan(8192, 1, regime=IT)
