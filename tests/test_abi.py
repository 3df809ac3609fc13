"""CPU-only checks of the boundary: the C-ABI library loads and exports every symbol
include/fif.h declares; host-side validation rejects bad plans without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "fif.h")).read()
    return sorted(set(re.findall(r"^\s*(?:fif_status|const char\*|int32_t)\s+(fif_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    import __graft_entry__ as ge

    ge.build_native()
    from paper_1802_01359_b200 import fif

    lib = fif.lib()
    decl = _header_symbols()
    assert len(decl) >= 13
    assert sorted(fif.SYMBOLS) == decl
    for name in decl:
        assert hasattr(lib, name), name


def test_status_strings():
    from paper_1802_01359_b200 import fif

    lib = fif.lib()
    for code, name in fif.STATUS.items():
        assert lib.fif_status_string(code).decode() == name


@pytest.mark.parametrize("args", [
    dict(n=8), dict(n=1023), dict(batch=-1), dict(xi=0.0), dict(delta=0.0), dict(delta=float("nan")),
    dict(max_inner=0), dict(max_imfs=0), dict(window=7), dict(dtype=5)])
def test_plan_validation_rejects_without_gpu(args):
    """Invalid arguments are refused on the host before any CUDA call (include/fif.h: INVALID_ARG /
    UNSUPPORTED_N, nothing enqueued)."""
    from paper_1802_01359_b200 import fif

    p = dict(n=1024, batch=4, dtype=0, window=0, xi=1.6, delta=1e-3, max_inner=200, max_imfs=10)
    p.update(args)
    h = ctypes.c_void_p()
    st = fif.lib().fif_plan_create(ctypes.byref(h), p["n"], p["batch"], p["dtype"], p["window"], p["xi"],
                                   p["delta"], p["max_inner"], p["max_imfs"])
    assert st in (1, 2) and not h.value


def test_unsupported_n_reported():
    from paper_1802_01359_b200 import fif

    h = ctypes.c_void_p()
    lib = fif.lib()
    for n in (7 * 1024, 2 * 11 * 512, 1 << 28, 3 << 27):  # not 2^a 3^b 5^c, or beyond n = 2^27
        assert lib.fif_plan_create(ctypes.byref(h), n, 1, 0, 0, 1.6, 1e-3, 200, 10) == 2, n
    assert lib.fif_plan_create_ex(ctypes.byref(h), 3 * 1024, 1, 0, 0, 1.6, 1e-3, 200, 10, 1) == 2  # not resident
    assert lib.fif_plan_create_ex(ctypes.byref(h), 1024, 1, 0, 0, 1.6, 1e-3, 200, 10, 9) == 1    # bad regime


def test_product_path_does_not_import_oracle():
    """The binding and the kernels never touch oracle/ (independence)."""
    pkg = os.path.join(ROOT, "paper_1802_01359_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "fif_oracle" not in src, f
