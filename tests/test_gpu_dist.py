"""GPU parity of the distributed regime (config 3: one long signal time-block sharded over P ranks).

On one GPU the P ranks run emulated (fif_plan_create_dist_emulated: every rank's kernels back to back,
the NCCL collectives replaced by device copies) -- the same kernels and the same static schedule the
NCCL plan runs, one rank per process.  Expected values come from the oracle (time-domain literal
iteration where it finishes in seconds, the paper's direct form oracle/direct_form.py otherwise)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import direct_form as df  # noqa: E402
from paper_1802_01359_b200 import fif, signals  # noqa: E402
from test_gpu_parity import TAU, assert_parity, run_gpu  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_native()
    torch.cuda.set_device(0)


def run_dist(s, P, dtype="f64", stop=fif.STOP_SD, gamma=0.0, **kw):
    """Decompose ONE signal s [n] with the emulated P-rank plan; returns the run_gpu layout for batch 1."""
    n = s.shape[0]
    plan = fif.Plan.dist(n, 0, P, dtype=dtype, emulated=True, **kw)
    if stop != fif.STOP_SD or gamma != 0.0:
        plan.set_options(stop, gamma)
    x = torch.from_numpy(np.ascontiguousarray(s.reshape(P, n // P))).cuda()
    imfs, count, lens, iters = plan.alloc_outputs()
    plan.decompose(x, imfs, count, lens, iters)
    torch.cuda.synchronize()
    imfs = imfs.cpu().numpy()  # [P][M+1][n/P]
    count, lens, iters = count.cpu().numpy(), lens.cpu().numpy(), iters.cpu().numpy()
    plan.close()
    # every rank reports the same integers
    assert (count == count[0]).all() and (lens == lens[0]).all() and (iters == iters[0]).all()
    full = np.concatenate([imfs[r] for r in range(P)], axis=1)[None]  # [1][M+1][n]
    return [full, count[:1], lens[:1], iters[:1]]


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_dist_emulated_vs_td_oracle(P):
    n = 4096
    for i in range(3):
        s = signals.tones_signal(n, 31, i)[None]
        gpu = run_dist(s[0], P)
        ref = oracle.decompose(s)
        assert_parity(s[0], gpu, ref, 0, 0)


@pytest.mark.parametrize("n,P", [(3 * 2048, 2), (3 * 2048, 4), (5 * 1024, 2)])
def test_dist_emulated_mixed_radix(n, P):
    s = signals.tones_signal(n, 32, 0)[None]
    gpu = run_dist(s[0], P)
    ref = oracle.decompose(s)
    assert_parity(s[0], gpu, ref, 0, 0)


def test_dist_degenerate_and_nonfinite():
    n, P = 2048, 4
    for s in (np.zeros(n), np.full(n, 2.5), np.linspace(-1.0, 1.0, n), np.cos(2 * np.pi * 40 * np.arange(n) / n + 0.1)):
        gpu = run_dist(s, P)
        ref = oracle.decompose(s[None])
        assert_parity(s, gpu, ref, 0, 0)
    bad = signals.tones_signal(n, 33, 0)
    bad[1500] = np.inf
    imfs, count, _, _ = run_dist(bad, P)
    assert count[0] == -1 and (imfs == 0).all()


def test_dist_parameters():
    n, P = 4096, 4
    s = signals.tones_signal(n, 34, 0)
    for kw in (dict(delta=1e-2, max_inner=50, max_imfs=3), dict(delta=0.3, max_inner=7, max_imfs=12)):
        gpu = run_dist(s, P, **kw)
        ref = oracle.decompose(s[None], **kw)
        assert_parity(s, gpu, ref, 0, 0)


def test_dist_fp32():
    n, P = 1 << 14, 4
    s32 = signals.cfg4_signal(n, 3)
    gpu = run_dist(s32, P, "f32")
    s64 = s32.astype(np.float64)
    ref = df.decompose_batch(s64[None], tau=TAU["f32"])
    assert_parity(s64, gpu, ref, 0, 0, "f32")


def test_dist_equals_single_gpu_streamed():
    n = 1 << 16
    s = signals.cfg3_signal(5, n=n)
    a = run_gpu(s[None], regime=fif.REGIME_STREAMED)
    for P in (2, 8):
        b = run_dist(s, P)
        np.testing.assert_array_equal(a[1], b[1])
        np.testing.assert_array_equal(a[2], b[2])
        np.testing.assert_array_equal(a[3], b[3])
        for m in range(a[1][0] + 1):
            x, y = a[0][0, m], b[0][0, m]
            assert np.linalg.norm(x - y) <= 1e-11 * max(np.linalg.norm(x), 1e-5 * np.linalg.norm(s))


def test_dist_cfg3_recipe_2p22_vs_direct_form():
    """cfg3 recipe at n = 2^22, 8 emulated ranks, against the paper's direct form."""
    n = 1 << 22
    s = signals.cfg3_signal(0, n=n)
    gpu = run_dist(s, 8)
    ref = df.decompose_batch(s[None])
    assert_parity(s, gpu, ref, 0, 0)


def test_dist_nccl_one_rank(monkeypatch):
    """The NCCL path itself (unique id, ncclCommInitRank, ncclAllGather, grouped ncclSend/ncclRecv -- to self)
    on the one GPU of this box: a one-rank plan forced through NCCL equals the single-GPU streamed plan."""
    monkeypatch.setenv("FIF_DIST_FORCE_NCCL", "1")
    n = 1 << 14
    s = signals.cfg3_signal(2, n=n)
    uid = fif.nccl_unique_id()
    assert len(uid) == 128
    plan = fif.Plan.dist(n, 0, 1, uid=uid)
    x = torch.from_numpy(s[None]).cuda()
    out = plan.alloc_outputs()
    plan.decompose(x, *out)
    torch.cuda.synchronize()
    b = [t.cpu().numpy() for t in out]
    plan.close()
    a = run_gpu(s[None], regime=fif.REGIME_STREAMED)
    for i in (1, 2, 3):
        np.testing.assert_array_equal(a[i], b[i])
    for m in range(a[1][0] + 1):
        assert np.linalg.norm(a[0][0, m] - b[0][0, m]) <= 1e-11 * max(np.linalg.norm(a[0][0, m]), 1e-5 * np.linalg.norm(s))


@pytest.mark.parametrize("P", [2, 4, 8])
def test_dist_peer_mode_fused_all_to_all(P, monkeypatch):
    """FIF_DIST_PEER: the four all-to-alls fused into their producing kernels as peer stores into the
    other ranks' buffers (NVLink in a multi-process plan; here the emulated ranks' buffers) -- same
    decomposition as the collective path and the oracle."""
    monkeypatch.setenv("FIF_DIST_PEER", "1")
    n = 4096
    for i in range(2):
        s = signals.tones_signal(n, 35, i)[None]
        gpu = run_dist(s[0], P)
        ref = oracle.decompose(s)
        assert_parity(s[0], gpu, ref, 0, 0)
    s = signals.cfg3_signal(7, n=1 << 16)
    monkeypatch.delenv("FIF_DIST_PEER")
    a = run_dist(s, P)
    monkeypatch.setenv("FIF_DIST_PEER", "1")
    b = run_dist(s, P)
    for i in (1, 2, 3):
        np.testing.assert_array_equal(a[i], b[i])
    assert np.abs(a[0] - b[0]).max() == 0.0  # the same arithmetic, only the data movement differs


def test_dist_peer_mode_nccl_one_rank(monkeypatch):
    """Peer mode through NCCL (IPC-handle all-gather + barrier all-reduce) on a one-rank communicator."""
    monkeypatch.setenv("FIF_DIST_FORCE_NCCL", "1")
    monkeypatch.setenv("FIF_DIST_PEER", "1")
    n = 1 << 14
    s = signals.cfg3_signal(3, n=n)
    plan = fif.Plan.dist(n, 0, 1, uid=fif.nccl_unique_id())
    x = torch.from_numpy(s[None]).cuda()
    out = plan.alloc_outputs()
    plan.decompose(x, *out)
    torch.cuda.synchronize()
    b = [t.cpu().numpy() for t in out]
    plan.close()
    a = run_gpu(s[None], regime=fif.REGIME_STREAMED)
    for i in (1, 2, 3):
        np.testing.assert_array_equal(a[i], b[i])
