"""GPU parity of the streamed regime (four-step FFT in HBM, kernel sequence per IMF): configs 2 and 4 and
mixed-radix lengths.  Same protocol as test_gpu_parity.py; where the literal time-domain oracle is too slow
(n >= 16384) the paper's direct form (oracle/direct_form.py, itself pinned to the time-domain oracle in
tests/test_oracle_pins.py) supplies the expected values."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import direct_form as df  # noqa: E402
from paper_1802_01359_b200 import fif, signals  # noqa: E402
from test_gpu_parity import TAU, assert_parity, df_batch, run_gpu, sample_idx  # noqa: E402

ST = fif.REGIME_STREAMED


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_native()
    torch.cuda.set_device(0)


@pytest.mark.parametrize("n", [1024, 4096])
def test_streamed_small_vs_td_oracle(n):
    s = np.stack([signals.tones_signal(n, 21, i) for i in range(6)])
    gpu = run_gpu(s, regime=ST)
    ref = oracle.decompose(s)
    for b in range(6):
        assert_parity(s[b], gpu, ref, b, b)


def test_streamed_equals_resident():
    s = signals.make_batch("cfg1", batch=64, start=500)
    a = run_gpu(s, regime=fif.REGIME_RESIDENT)
    b = run_gpu(s, regime=ST)
    np.testing.assert_array_equal(a[1], b[1])
    np.testing.assert_array_equal(a[2], b[2])
    np.testing.assert_array_equal(a[3], b[3])
    for i in range(64):
        for m in range(a[1][i] + 1):
            x, y = a[0][i, m], b[0][i, m]
            assert np.linalg.norm(x - y) <= 1e-11 * max(np.linalg.norm(x), 1e-5 * np.linalg.norm(s[i]))


@pytest.mark.parametrize("n", [3 * 1024, 5 * 1024, 3 * 512 * 5])
def test_streamed_mixed_radix_vs_td_oracle(n):
    s = np.stack([signals.tones_signal(n, 22, i) for i in range(4)])
    gpu = run_gpu(s, regime=ST)
    ref = oracle.decompose(s)
    for b in range(4):
        assert_parity(s[b], gpu, ref, b, b)


def test_cfg2_full_batch_sampled():
    """Config 2 at full size (512 x 65536 fp64, delta = 1e-4, the bench launch): every (B/64)-th signal (65)
    vs the direct form (spread over the host's cores), all compared in full; telescoping on every signal."""
    B = 512
    s = signals.make_batch("cfg2", batch=B)
    gpu = run_gpu(s, delta=1e-4)
    idx = sample_idx(B)
    ref = df_batch(s[idx], delta=1e-4)
    for i, b in enumerate(idx):
        assert_parity(s[b], gpu, ref, b, i)
    imfs, count = gpu[0], gpu[1]
    assert ((count >= 1) & (count <= 10)).all()
    assert np.abs(imfs.sum(axis=1) - s).max() <= 1e-11 * np.abs(s).max()


@pytest.mark.parity(min_full=0.1)  # fp32: see tests/test_gpu_parity.py::test_fp32_path
@pytest.mark.parametrize("n", [1 << 14, 1 << 17, 3 << 14, 5 << 14])
def test_cfg4_fp32_lengths(n):
    B = 6
    s32 = np.stack([signals.cfg4_signal(n, i) for i in range(B)])
    gpu = run_gpu(s32, "f32")
    s64 = s32.astype(np.float64)
    ref = df.decompose_batch(s64, tau=TAU["f32"])
    for b in range(B):
        assert_parity(s64[b], gpu, ref, b, b, "f32")


@pytest.mark.parity(min_full=0.1)  # fp32: see tests/test_gpu_parity.py::test_fp32_path
def test_cfg4_fp32_2p20():
    n, B = 1 << 20, 8
    s32 = np.stack([signals.cfg4_signal(n, i) for i in range(B)])
    gpu = run_gpu(s32, "f32")
    s64 = s32.astype(np.float64)
    ref = df_batch(s64, tau=TAU["f32"])
    for b in range(B):
        assert_parity(s64[b], gpu, ref, b, b, "f32")


def test_streamed_degenerate_and_nonfinite():
    n = 3 * 1024
    rows = [np.zeros(n), np.full(n, 1.5), np.linspace(-1, 1, n), signals.tones_signal(n, 23, 0),
            np.cos(2 * np.pi * 48 * np.arange(n) / n + 0.2)]
    s = np.stack(rows)
    s_bad = s.copy()
    s_bad[3, 7] = np.nan
    gpu = run_gpu(s, regime=ST)
    ref = oracle.decompose(s)
    for b in range(len(rows)):
        assert_parity(s[b], gpu, ref, b, b)
    bad = run_gpu(s_bad, regime=ST)
    assert bad[1][3] == -1 and (bad[0][3] == 0).all()
    assert_parity(s[4], bad, ref, 4, 4)


def test_streamed_parameters():
    s = np.stack([signals.tones_signal(2048, 24, i) for i in range(4)])
    for kw in (dict(delta=1e-2, max_inner=50, max_imfs=3), dict(delta=0.3, max_inner=7, max_imfs=12),
               dict(delta=1e-3, max_inner=1, max_imfs=4)):
        gpu = run_gpu(s, regime=ST, **kw)
        ref = oracle.decompose(s, **kw)
        for b in range(4):
            assert_parity(s[b], gpu, ref, b, b)


def test_streamed_host_path():
    s = np.stack([signals.tones_signal(5 * 1024, 25, i) for i in range(40)])
    dev = run_gpu(s)
    plan = fif.Plan(5 * 1024, 40, "f64")
    assert plan.launch_config()["regime"] == "streamed"
    hs = torch.from_numpy(s).pin_memory()
    outs = [torch.empty(tuple(t.shape), dtype=t.dtype).pin_memory() for t in plan.alloc_outputs("cpu")]
    plan.decompose_host(hs, *outs)
    for a, b in zip(dev, outs):
        np.testing.assert_array_equal(a, b.numpy())
    plan.close()


@pytest.mark.parametrize("n,rowmax,colmax", [(4096, 16, 16), (4096, 16, 8), (15360, 30, 16), (3 << 12, 24, 8)])
def test_streamed_multilevel_vs_td_oracle(n, rowmax, colmax, monkeypatch):
    """3- and 4-level geometries (forced by capping the level lengths) against the literal oracle."""
    monkeypatch.setenv("FIF_ST_ROWMAX", str(rowmax))
    monkeypatch.setenv("FIF_ST_COLMAX", str(colmax))
    s = np.stack([signals.tones_signal(n, 26, i) for i in range(3)])
    gpu = run_gpu(s, regime=ST)
    ref = oracle.decompose(s)
    for b in range(3):
        assert_parity(s[b], gpu, ref, b, b)


def test_streamed_long_single_signal_3level():
    """One cfg3-recipe signal of n = 2^23 (3-level geometry, batch 1) against the direct form."""
    n = 1 << 23
    s = signals.cfg3_signal(0, n=n)[None, :]
    gpu = run_gpu(s)
    ref = df.decompose_batch(s)
    assert_parity(s[0], gpu, ref, 0, 0)
    assert np.abs(gpu[0][0].sum(axis=0) - s[0]).max() <= 1e-11 * np.abs(s).max()


def test_streamed_many_waves_two_streams(monkeypatch):
    """L2 waves (FIF_WAVE_MB forces ~2 signals per wave, alternating between the plan's two streams) give
    the same decomposition as the resident regime, including signals that need the K-ary search."""
    monkeypatch.setenv("FIF_WAVE_MB", "0.2")
    s = signals.make_batch("cfg1", batch=41, start=900)  # ragged last wave
    a = run_gpu(s, regime=fif.REGIME_RESIDENT)
    b = run_gpu(s, regime=ST)
    assert (a[3] < 200).any()  # some IMFs stop below the cap (search + redo path)
    np.testing.assert_array_equal(a[1], b[1])
    np.testing.assert_array_equal(a[2], b[2])
    np.testing.assert_array_equal(a[3], b[3])
    for i in range(41):
        for m in range(a[1][i] + 1):
            x, y = a[0][i, m], b[0][i, m]
            assert np.linalg.norm(x - y) <= 1e-11 * max(np.linalg.norm(x), 1e-5 * np.linalg.norm(s[i]))


@pytest.mark.parametrize("n", [16, 24, 40, 96, 250])
def test_streamed_tiny_lengths_vs_td_oracle(n):
    """Smallest geometries (two levels of 2..5-point DFTs, self-paired rows only) against the literal oracle."""
    rng = np.random.default_rng(n)
    s = rng.standard_normal((5, n))
    gpu = run_gpu(s, regime=ST)
    ref = oracle.decompose(s)
    for b in range(5):
        assert_parity(s[b], gpu, ref, b, b)


def test_streamed_empty_batch():
    plan = fif.Plan(1 << 14, 0, "f64")
    x = torch.empty((0, 1 << 14), dtype=torch.float64, device="cuda")
    out = plan.alloc_outputs()
    plan.decompose(x, *out)  # a no-op
    torch.cuda.synchronize()
    plan.close()


@pytest.mark.parametrize("n,dtype,rowmax,colmax", [(1 << 17, "f64", None, None), (1 << 14, "f64", 64, 64),
                                                   (1 << 17, "f32", None, None), (3 << 14, "f32", None, None),
                                                   (5 << 14, "f32", None, None), (1 << 20, "f32", None, None)])
@pytest.mark.parametrize("mode", ["1", "2"])
def test_streamed_bulk_copy_tiles_bit_identical(n, dtype, rowmax, colmax, mode, monkeypatch):
    """The column tiles staged by the TMA engine (row-major; FIF_ST_RM=1: one cp.async.bulk per tile row,
    FIF_ST_RM=2: one cp.async.bulk.tensor box per tile from a per-call tensor map) run the same butterflies in the
    same order as the default cp.async tiles: identical decompositions, bit for bit (2-, 3-level, mixed-radix
    geometries; both dtypes)."""
    if rowmax:
        monkeypatch.setenv("FIF_ST_ROWMAX", str(rowmax))
        monkeypatch.setenv("FIF_ST_COLMAX", str(colmax))
    B = 3
    s = (np.stack([signals.cfg4_signal(n, i) for i in range(B)]) if dtype == "f32"
         else np.stack([signals.tones_signal(n, 27, i) for i in range(B)]))
    monkeypatch.setenv("FIF_ST_RM", "0")  # the cp.async tiles (the default is the tensor-map tiles, mode 2)
    a = run_gpu(s, dtype, regime=ST)
    monkeypatch.setenv("FIF_ST_RM", mode)
    b = run_gpu(s, dtype, regime=ST)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
