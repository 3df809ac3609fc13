"""Thin Python binding of the C ABI in include/fif.h (argument marshalling only).

Every step of the decomposition runs in the sm_100a kernels of libfif_b200.so;
this module only passes pointers, sizes and streams.  PyTorch is used for
device memory and streams.  There is no CPU fallback: if the shared library is
missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FIF_LIB_PATH", os.path.join(_HERE, "libfif_b200.so"))  # override: dev A/B builds

F64, F32 = 0, 1
WINDOW_TRI_SQ, WINDOW_TRI_SQ_WIDE = 0, 1
STATUS = {0: "FIF_OK", 1: "FIF_ERR_INVALID_ARG", 2: "FIF_ERR_UNSUPPORTED_N", 3: "FIF_ERR_OOM", 4: "FIF_ERR_CUDA",
          5: "FIF_ERR_NCCL"}

# every symbol include/fif.h declares (checked by tests/test_abi.py)
REGIME_AUTO, REGIME_RESIDENT, REGIME_STREAMED, REGIME_ITERATIVE, REGIME_CLUSTER = 0, 1, 2, 3, 4
SYMBOLS = ["fif_plan_create", "fif_plan_create_ex", "fif_decompose", "fif_decompose_host", "fif_destroy", "fif_status_string",
           "fif_plan_kernels_per_call", "fif_plan_regime", "fif_plan_launch_config", "fif_test_rfft",
           "fif_test_irfft", "fif_test_extrema", "fif_test_window_spectrum", "fif_test_inner", "fif_nccl_unique_id",
           "fif_plan_create_dist", "fif_plan_create_dist_emulated", "fif_plan_set_options", "fif_plan_set_mask_rule",
           "fif_plan_workspace_bytes", "fif_plan_set_workspace", "fif_plan_set_eigen_table"]
STOP_SD, STOP_N0 = 0, 1
MASK_EXTREMA, MASK_SPECTRAL = 0, 1


class FifError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {STATUS.get(status, status)}")
        self.status = status


_lib = None


def lib():
    """Load libfif_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FifError(-1, f"native library missing ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32)
        i64, i32, d = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.fif_plan_create.argtypes = [ctypes.POINTER(vp), i64, i64, ctypes.c_int, ctypes.c_int, d, d, i32, i32]
        L.fif_plan_create_ex.argtypes = [ctypes.POINTER(vp), i64, i64, ctypes.c_int, ctypes.c_int, d, d, i32, i32,
                                         ctypes.c_int]
        L.fif_decompose.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.fif_decompose_host.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.fif_destroy.argtypes = [vp]
        L.fif_status_string.argtypes = [ctypes.c_int]
        L.fif_status_string.restype = ctypes.c_char_p
        L.fif_plan_kernels_per_call.argtypes = [vp]
        L.fif_plan_kernels_per_call.restype = i32
        L.fif_plan_regime.argtypes = [vp]
        L.fif_plan_regime.restype = ctypes.c_char_p
        L.fif_plan_launch_config.argtypes = [vp, i32p, i32p, i32p]
        L.fif_test_rfft.argtypes = [vp, i64, vp, vp, vp]
        L.fif_test_irfft.argtypes = [vp, i64, vp, vp, vp]
        L.fif_test_extrema.argtypes = [vp, i64, vp, vp, vp]
        L.fif_test_window_spectrum.argtypes = [vp, i32, vp, vp]
        L.fif_test_inner.argtypes = [vp, i64, i32, vp, vp, vp, vp]
        L.fif_nccl_unique_id.argtypes = [vp]
        L.fif_plan_set_options.argtypes = [vp, ctypes.c_int, d]
        L.fif_plan_set_mask_rule.argtypes = [vp, ctypes.c_int]
        L.fif_plan_workspace_bytes.argtypes = [vp, ctypes.POINTER(ctypes.c_size_t)]
        L.fif_plan_set_workspace.argtypes = [vp, vp, ctypes.c_size_t]
        L.fif_plan_set_eigen_table.argtypes = [vp, i32]
        L.fif_plan_create_dist.argtypes = [ctypes.POINTER(vp), i64, ctypes.c_int, ctypes.c_int, d, d, i32, i32, vp,
                                           i32, i32]
        L.fif_plan_create_dist_emulated.argtypes = [ctypes.POINTER(vp), i64, ctypes.c_int, ctypes.c_int, d, d, i32,
                                                    i32, i32]
        for name in SYMBOLS:
            if name not in ("fif_status_string", "fif_plan_kernels_per_call", "fif_plan_regime"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(st: int, what: str):
    if st != 0:
        raise FifError(st, what)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream_ptr(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def nccl_unique_id() -> bytes:
    """fif_nccl_unique_id: 128 bytes for fif_plan_create_dist (call on rank 0, broadcast)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().fif_nccl_unique_id(buf), "fif_nccl_unique_id")
    return buf.raw


class Plan:
    """fif_plan_create(n, batch, dtype, window, xi, delta, max_inner, max_imfs)."""

    def __init__(self, n, batch, dtype="f64", window=WINDOW_TRI_SQ, xi=1.6, delta=1e-3, max_inner=200,
                 max_imfs=10, regime=REGIME_AUTO):
        self.n, self.batch, self.max_imfs = int(n), int(batch), int(max_imfs)
        self.dtype = dtype
        self._h = ctypes.c_void_p()
        _check(lib().fif_plan_create_ex(ctypes.byref(self._h), self.n, self.batch, F64 if dtype == "f64" else F32,
                                        int(window), float(xi), float(delta), int(max_inner), int(max_imfs),
                                        int(regime)), "fif_plan_create_ex")

    @property
    def handle(self):
        return self._h

    def torch_dtype(self):
        import torch
        return torch.float64 if self.dtype == "f64" else torch.float32

    def alloc_outputs(self, device="cuda"):
        import torch
        imfs = torch.empty((self.batch, self.max_imfs + 1, self.n), dtype=self.torch_dtype(), device=device)
        count = torch.empty(self.batch, dtype=torch.int32, device=device)
        lens = torch.empty((self.batch, self.max_imfs), dtype=torch.int32, device=device)
        iters = torch.empty((self.batch, self.max_imfs), dtype=torch.int32, device=device)
        return imfs, count, lens, iters

    def set_options(self, stop=STOP_SD, gamma=0.0):
        """fif_plan_set_options: stopping rule (STOP_SD / STOP_N0) and gamma-threshold (0 = off)."""
        _check(lib().fif_plan_set_options(self._h, int(stop), float(gamma)), "fif_plan_set_options")
        return self

    def set_mask_rule(self, rule=MASK_EXTREMA):
        """fif_plan_set_mask_rule: filter length from the extrema count or the highest spectral peak."""
        _check(lib().fif_plan_set_mask_rule(self._h, int(rule)), "fif_plan_set_mask_rule")
        return self

    def set_eigen_table(self, enable=True):
        """fif_plan_set_eigen_table: precompute w_hat for every L (resident regime), or free it."""
        _check(lib().fif_plan_set_eigen_table(self._h, int(bool(enable))), "fif_plan_set_eigen_table")
        return self

    def workspace_bytes(self):
        """fif_plan_workspace_bytes: device scratch the plan's decompose needs (0: none)."""
        b = ctypes.c_size_t()
        _check(lib().fif_plan_workspace_bytes(self._h, ctypes.byref(b)), "fif_plan_workspace_bytes")
        return int(b.value)

    def set_workspace(self, ws=None):
        """fif_plan_set_workspace: hand the plan a caller-owned device buffer (a uint8 torch tensor of at
        least workspace_bytes(), 256-byte aligned); None returns to a plan-owned workspace.  The tensor is
        kept referenced here so it outlives its use."""
        _check(lib().fif_plan_set_workspace(self._h, _ptr(ws), ctypes.c_size_t(0 if ws is None else ws.numel()
                                                                                * ws.element_size())),
               "fif_plan_set_workspace")
        self._ws = ws
        return self

    def decompose(self, signals, imfs, count, lens, iters, stream=None):
        """fif_decompose on device tensors (asynchronous on `stream`)."""
        _check(lib().fif_decompose(self._h, _ptr(signals), _ptr(imfs), _ptr(count), _ptr(lens), _ptr(iters),
                                   _stream_ptr(stream)), "fif_decompose")

    def decompose_host(self, signals, imfs, count, lens, iters, stream=None):
        """fif_decompose_host on (pinned) host tensors; synchronous."""
        _check(lib().fif_decompose_host(self._h, _ptr(signals), _ptr(imfs), _ptr(count), _ptr(lens), _ptr(iters),
                                        _stream_ptr(stream)), "fif_decompose_host")

    @classmethod
    def dist(cls, n_global, rank, nranks, uid=None, dtype="f64", window=WINDOW_TRI_SQ, xi=1.6, delta=1e-3,
             max_inner=200, max_imfs=10, emulated=False):
        """fif_plan_create_dist (one rank of nranks; uid = nccl_unique_id() of rank 0) or, with
        emulated=True, fif_plan_create_dist_emulated (all nranks ranks on this device)."""
        self = cls.__new__(cls)
        self.n, self.max_imfs, self.dtype = int(n_global) // int(nranks), int(max_imfs), dtype
        self.batch = int(nranks) if emulated else 1
        self._h = ctypes.c_void_p()
        dt = F64 if dtype == "f64" else F32
        if emulated:
            _check(lib().fif_plan_create_dist_emulated(ctypes.byref(self._h), int(n_global), dt, int(window),
                                                       float(xi), float(delta), int(max_inner), int(max_imfs),
                                                       int(nranks)), "fif_plan_create_dist_emulated")
        else:
            ub = ctypes.create_string_buffer(bytes(uid) if uid is not None else bytes(128), 128)
            _check(lib().fif_plan_create_dist(ctypes.byref(self._h), int(n_global), dt, int(window), float(xi),
                                              float(delta), int(max_inner), int(max_imfs), ub, int(rank),
                                              int(nranks)), "fif_plan_create_dist")
        return self

    def launch_config(self):
        g, b, s = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().fif_plan_launch_config(self._h, ctypes.byref(g), ctypes.byref(b), ctypes.byref(s)),
               "fif_plan_launch_config")
        return {"grid": g.value, "block": b.value, "smem": s.value, "regime": lib().fif_plan_regime(self._h).decode(),
                "kernels_per_call": lib().fif_plan_kernels_per_call(self._h)}

    # test hooks ---------------------------------------------------------------------------------
    def test_rfft(self, x, out, stream=None):
        _check(lib().fif_test_rfft(self._h, x.shape[0], _ptr(x), _ptr(out), _stream_ptr(stream)), "fif_test_rfft")

    def test_irfft(self, X, out, stream=None):
        _check(lib().fif_test_irfft(self._h, X.shape[0], _ptr(X), _ptr(out), _stream_ptr(stream)), "fif_test_irfft")

    def test_extrema(self, x, k, stream=None):
        _check(lib().fif_test_extrema(self._h, x.shape[0], _ptr(x), _ptr(k), _stream_ptr(stream)), "fif_test_extrema")

    def test_window_spectrum(self, L, out, stream=None):
        _check(lib().fif_test_window_spectrum(self._h, int(L), _ptr(out), _stream_ptr(stream)),
               "fif_test_window_spectrum")

    def test_inner(self, L, x, imf, N, stream=None):
        _check(lib().fif_test_inner(self._h, x.shape[0], int(L), _ptr(x), _ptr(imf), _ptr(N), _stream_ptr(stream)),
               "fif_test_inner")

    def close(self):
        if self._h:
            lib().fif_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decompose(signals, window=WINDOW_TRI_SQ, xi=1.6, delta=1e-3, max_inner=200, max_imfs=10, stream=None):
    """Convenience: decompose a CUDA tensor [B, n] (f64 or f32); returns (imfs, count, lens, iters)."""
    import torch
    assert signals.is_cuda and signals.dim() == 2
    dtype = "f64" if signals.dtype == torch.float64 else "f32"
    plan = Plan(signals.shape[1], signals.shape[0], dtype, window, xi, delta, max_inner, max_imfs)
    out = plan.alloc_outputs(signals.device)
    plan.decompose(signals.contiguous(), *out, stream=stream)
    torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
    plan.close()
    return out
