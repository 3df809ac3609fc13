"""Race / schedule checks (compute-sanitizer is closed on this pool: DESIGN.md §5): every regime's kernels
must produce the SAME BITS whatever the CTA schedule -- repeated runs, and persistent grids capped to a few
CTAs (FIF_GRID_CAP, read at plan creation), which changes which CTA handles which signal / tile / unit and
how the last-CTA-decides reductions interleave.  A missing barrier, a shared-memory race or an
order-dependent reduction shows up as a bit difference here."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1802_01359_b200 import fif, signals  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_native()
    torch.cuda.set_device(0)


def _run(make_plan, s, monkeypatch, cap=None):
    if cap:
        monkeypatch.setenv("FIF_GRID_CAP", str(cap))
    else:
        monkeypatch.delenv("FIF_GRID_CAP", raising=False)
    plan = make_plan()
    monkeypatch.delenv("FIF_GRID_CAP", raising=False)
    x = torch.from_numpy(np.ascontiguousarray(s)).cuda()
    out = plan.alloc_outputs()
    plan.decompose(x, *out)
    torch.cuda.synchronize()
    res = [t.cpu().numpy().copy() for t in out]
    plan.close()
    return res


def _same(a, b):
    for x, y in zip(a, b):
        assert x.tobytes() == y.tobytes()


@pytest.mark.parametrize("case", ["resident", "resident_table", "resident_f32", "streamed", "streamed_mixed",
                                  "distributed", "distributed_peer"])
def test_bits_independent_of_schedule(case, monkeypatch):
    if case.startswith("resident"):
        dt = "f32" if case.endswith("f32") else "f64"
        s = signals.make_batch("cfg1", batch=40, n=1024) if dt == "f64" else \
            np.stack([signals.cfg4_signal(1024, i) for i in range(40)])

        def mk():
            p = fif.Plan(1024, 40, dt)
            if case == "resident_table":
                p.set_eigen_table(True)
            return p
    elif case.startswith("streamed"):
        n = 4096 if case == "streamed" else 3 * 1024
        s = np.stack([signals.tones_signal(n, 31, i) for i in range(5)])

        def mk():
            return fif.Plan(n, 5, "f64", regime=fif.REGIME_STREAMED)
    else:
        if case == "distributed_peer":
            monkeypatch.setenv("FIF_DIST_PEER", "1")
        n = 1 << 15
        s = signals.cfg3_signal(0, n=n).reshape(4, -1)

        def mk():
            return fif.Plan.dist(n, 0, 4, emulated=True)
    ref = _run(mk, s, monkeypatch)
    _same(ref, _run(mk, s, monkeypatch))          # repeated run
    for cap in (1, 3, 7):                          # other CTA schedules
        _same(ref, _run(mk, s, monkeypatch, cap))
