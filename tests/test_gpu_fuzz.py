"""Seeded randomised parity sweep: plan shapes and parameters drawn at random over the supported space
(length -- power-of-two and mixed-radix, resident and streamed, forced 3-level geometries --, batch,
dtype, window, delta, max_inner, max_imfs, the method options, the per-L table), each decomposition
against the paper's direct form (oracle/direct_form.py, pinned to the time-domain oracle in
tests/test_oracle_pins.py) with the protocol of test_gpu_parity.py."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import direct_form as df  # noqa: E402
from paper_1802_01359_b200 import fif, signals  # noqa: E402
from test_gpu_parity import TAU, assert_parity  # noqa: E402

LENGTHS = [512, 1024, 2048, 4096, 8192, 3 * 1024, 5 * 1024, 3 * 5 * 512, 9 * 1024, 16384, 25 * 512, 3 * 8192]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_native()
    torch.cuda.set_device(0)


def _case(seed):
    rng = np.random.default_rng([20261020, seed])
    n = int(rng.choice(LENGTHS))
    pow2 = (n & (n - 1)) == 0
    dtype = "f32" if rng.random() < 0.3 else "f64"
    regime = fif.REGIME_AUTO
    if pow2 and n <= 8192 and rng.random() < 0.4:
        regime = fif.REGIME_STREAMED
    p = dict(n=n, B=int(rng.integers(1, 7)), dtype=dtype, regime=regime,
             window=int(rng.random() < 0.25), delta=float(10 ** rng.uniform(-4, -1.5)),
             max_inner=int(rng.choice([1, 7, 50, 200, 333])), max_imfs=int(rng.integers(1, 12)),
             stop=fif.STOP_SD, gamma=0.0, mask=fif.MASK_EXTREMA, eig=False, levels3=False)
    u = rng.random()
    if u < 0.12:
        p["gamma"] = float(rng.uniform(0.01, 0.3))
    elif u < 0.22:
        p["mask"] = fif.MASK_SPECTRAL
    elif u < 0.3:
        p["stop"], p["delta"] = fif.STOP_N0, float(rng.uniform(2.0, 30.0))
    p["eig"] = rng.random() < 0.4
    p["levels3"] = regime == fif.REGIME_STREAMED and rng.random() < 0.3
    p["sig_seed"] = int(rng.integers(0, 1 << 30))
    return p


# random shapes and parameters (fp32, max_inner = 1, small delta ...) produce decisions at the oracle's margin
# thresholds by construction: fp64 cases compare every signal on at least its first IMF (in full when safe);
# fp32 cases whatever the margins allow (a first SD decision within the fp32 threshold is common)
def _fuzz_floor(request, dtype):
    request.node.add_marker(pytest.mark.parity(min_full=0.0, min_prefix=1 if dtype == "f64" else 0))


@pytest.mark.parametrize("seed", range(int(os.environ.get("FIF_FUZZ_CASES", "40"))))
def test_fuzz_vs_direct_form(seed, monkeypatch, request):
    p = _case(seed)
    _fuzz_floor(request, p["dtype"])
    n, B = p["n"], p["B"]
    s = np.stack([signals.tones_signal(n, 77, p["sig_seed"] + i) for i in range(B)])
    if p["dtype"] == "f32":
        s = s.astype(np.float32)
    if p["levels3"]:  # force a deeper multi-level geometry at this small n (test-only knobs, read at create)
        monkeypatch.setenv("FIF_ST_ROWMAX", "64")
        monkeypatch.setenv("FIF_ST_COLMAX", "16")
    plan = fif.Plan(n, B, p["dtype"], window=p["window"], delta=p["delta"], max_inner=p["max_inner"],
                    max_imfs=p["max_imfs"], regime=p["regime"])
    monkeypatch.delenv("FIF_ST_ROWMAX", raising=False)
    monkeypatch.delenv("FIF_ST_COLMAX", raising=False)
    plan.set_options(p["stop"], p["gamma"]).set_mask_rule(p["mask"])
    if p["eig"] and plan.launch_config()["regime"] == "resident":
        plan.set_eigen_table(True)
    x = torch.from_numpy(np.ascontiguousarray(s)).cuda()
    out = plan.alloc_outputs()
    plan.decompose(x, *out)
    torch.cuda.synchronize()
    gpu = [t.cpu().numpy() for t in out]
    plan.close()
    s64 = s.astype(np.float64)
    ref = df.decompose_batch(s64, delta=p["delta"], max_inner=p["max_inner"], max_imfs=p["max_imfs"],
                             window=p["window"], gamma=p["gamma"], stop=p["stop"], mask=p["mask"],
                             tau=TAU[p["dtype"]])
    for b in range(B):
        assert_parity(s64[b], gpu, ref, b, b, p["dtype"])


@pytest.mark.parametrize("seed", range(int(os.environ.get("FIF_FUZZ_DIST_CASES", "12"))))
def test_fuzz_distributed_vs_direct_form(seed, request):
    """One signal over P emulated ranks (the distributed regime): random P, length, dtype, window,
    parameters and stopping options."""
    from test_gpu_dist import run_dist

    rng = np.random.default_rng([20261021, seed])
    P = int(rng.choice([1, 2, 4, 8]))
    n = int(rng.choice([4096, 8192, 16384, 3 * 4096 * 2, 5 * 4096]))
    if (n // 2) % (P * P):
        P = 2
    dtype = "f32" if rng.random() < 0.3 else "f64"
    kw = dict(window=int(rng.random() < 0.25), delta=float(10 ** rng.uniform(-4, -1.5)),
              max_inner=int(rng.choice([1, 9, 200])), max_imfs=int(rng.integers(1, 11)))
    stop, gamma = fif.STOP_SD, 0.0
    u = rng.random()
    if u < 0.15:
        gamma = float(rng.uniform(0.01, 0.3))
    elif u < 0.3:
        stop, kw["delta"] = fif.STOP_N0, float(rng.uniform(2.0, 30.0))
    s = signals.tones_signal(n, 78, int(rng.integers(0, 1 << 30)))
    if dtype == "f32":
        s = s.astype(np.float32)
    _fuzz_floor(request, dtype)
    plan_kw = dict(kw)
    gpu = run_dist(s, P, dtype=dtype, stop=stop, gamma=gamma, **plan_kw)
    s64 = s.astype(np.float64)[None]
    ref = df.decompose_batch(s64, gamma=gamma, stop=stop, tau=TAU[dtype], **kw)
    assert_parity(s64[0], gpu, ref, 0, 0, dtype)
