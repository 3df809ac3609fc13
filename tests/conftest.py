import math
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# Every GPU parity comparison (test_gpu_parity.assert_parity) records (prefix P, full, M) here; the autouse
# fixture below then enforces the test's floor: by default EVERY compared signal must be compared in full
# (all its decisions safe by the oracle's margins, reading A21); a test whose inputs legitimately carry
# unsafe decisions states its floor with @pytest.mark.parity(min_full=..., min_prefix=...) -- the fraction
# of signals compared in full and the smallest number of leading IMFs compared on any signal.
PARITY_LOG = []


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running oracle checks")
    config.addinivalue_line("markers", "parity(min_full=1.0, min_prefix=0): the test's parity floor (conftest.py)")


@pytest.fixture(autouse=True)
def _parity_floor(request):
    PARITY_LOG.clear()
    yield
    if not PARITY_LOG:
        return
    mk = request.node.get_closest_marker("parity")
    min_full = mk.kwargs.get("min_full", 1.0) if mk else 1.0
    min_prefix = mk.kwargs.get("min_prefix", 0) if mk else 0
    n = len(PARITY_LOG)
    nfull = sum(1 for _, full, _ in PARITY_LOG if full)
    assert nfull >= math.ceil(min_full * n - 1e-9), \
        f"parity floor: {nfull}/{n} signals compared in full, the test requires >= {min_full:.2f}"
    partial = [p for p, full, _ in PARITY_LOG if not full]
    worst = min(partial) if partial else None
    assert worst is None or worst >= min_prefix, \
        f"parity floor: a signal compared on {worst} leading IMFs only (< {min_prefix})"
    print(f"[parity] {nfull}/{n} signals in full, shortest partial prefix {worst}")
