"""Caller-owned decompose workspace (include/fif.h fif_plan_workspace_bytes / fif_plan_set_workspace;
SURVEY.md §8b "ownership"): a streamed plan run in a caller buffer (torch-allocated, pre-filled with
garbage) gives bit-identical outputs to the plan-owned workspace -- whose results the parity tests pin
to the oracle -- and every misuse is refused."""
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


def _run(plan, x):
    out = plan.alloc_outputs()
    plan.decompose(x, *out)
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in out]


def _same(a, b):
    for u, v in zip(a, b):
        np.testing.assert_array_equal(u, v)


def _garbage(nbytes, offset=0):
    t = torch.empty(nbytes + 512, dtype=torch.uint8, device="cuda")
    t.fill_(0xA5)
    base = (256 - t.data_ptr() % 256) % 256 + offset
    return t[base:base + nbytes]


@pytest.mark.parametrize("n,dtype", [(16384, "f64"), (3 * 4096, "f32")])
def test_caller_workspace_bit_identical(n, dtype):
    s = np.stack([signals.tones_signal(n, 31, i) for i in range(5)])
    x = torch.from_numpy(s).to(torch.float64 if dtype == "f64" else torch.float32).cuda()
    plan = fif.Plan(n, 5, dtype, regime=fif.REGIME_STREAMED)
    need = plan.workspace_bytes()
    assert need >= 2 * 5 * (n // 2) * (16 if dtype == "f64" else 8)
    ref = _run(plan, x)
    plan.set_workspace(_garbage(need))
    _same(ref, _run(plan, x))
    _same(ref, _run(plan, x))          # the control state left by a call is valid for the next
    plan.set_workspace(None)           # back to a plan-owned workspace
    _same(ref, _run(plan, x))


def test_workspace_misuse_refused():
    n = 8192 * 2
    plan = fif.Plan(n, 3, "f64", regime=fif.REGIME_STREAMED)
    need = plan.workspace_bytes()
    lib = fif.lib()
    small = _garbage(need - 256)
    assert lib.fif_plan_set_workspace(plan.handle, fif._ptr(small), need - 256) == 1
    mis = _garbage(need, offset=8)
    assert lib.fif_plan_set_workspace(plan.handle, fif._ptr(mis), need) == 1
    host = torch.empty(need + 256, dtype=torch.uint8).pin_memory()
    hp = host.data_ptr() + (256 - host.data_ptr() % 256) % 256
    import ctypes
    assert lib.fif_plan_set_workspace(plan.handle, ctypes.c_void_p(hp), need) == 1
    # the plan still works on its own workspace after the refusals
    s = np.stack([signals.tones_signal(n, 32, i) for i in range(3)])
    x = torch.from_numpy(s).cuda()
    a = _run(plan, x)
    b = _run(fif.Plan(n, 3, "f64", regime=fif.REGIME_STREAMED), x)
    _same(a, b)


def test_mask_rule_with_caller_workspace():
    n = 16384
    s = np.stack([signals.tones_signal(n, 33, i) for i in range(4)])
    x = torch.from_numpy(s).cuda()
    own = fif.Plan(n, 4, "f64", regime=fif.REGIME_STREAMED)
    base = own.workspace_bytes()
    own.set_mask_rule(fif.MASK_SPECTRAL)
    need = own.workspace_bytes()
    assert need > base
    ref_spec = _run(own, x)
    plan = fif.Plan(n, 4, "f64", regime=fif.REGIME_STREAMED).set_workspace(_garbage(base))
    ref_ext = _run(plan, x)
    with pytest.raises(fif.FifError):      # caller workspace too small for the power array: refused
        plan.set_mask_rule(fif.MASK_SPECTRAL)
    _same(ref_ext, _run(plan, x))          # rule unchanged
    plan.set_workspace(_garbage(need)).set_mask_rule(fif.MASK_SPECTRAL)
    _same(ref_spec, _run(plan, x))
    plan.set_mask_rule(fif.MASK_EXTREMA)
    _same(ref_ext, _run(plan, x))


def test_resident_and_distributed_workspace():
    res = fif.Plan(4096, 2, "f64")
    assert res.workspace_bytes() == 0
    res.set_workspace(_garbage(1024))     # no-op
    d = fif.Plan.dist(1 << 16, 0, 2, None, emulated=True)
    assert d.workspace_bytes() == 0
    assert fif.lib().fif_plan_set_workspace(d.handle, fif._ptr(_garbage(1 << 20)), 1 << 20) == 1
