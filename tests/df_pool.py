"""Test infrastructure: runs oracle/direct_form.py over independent signals in separate host processes
('spawn': the workers import only numpy and the oracle, never torch or CUDA).  Not product code."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _one(args):
    from oracle import direct_form as df

    row, kw = args
    return df.decompose(row, **kw)


def df_batch(signals_, **kw):
    """oracle/direct_form.decompose on each row (the oracle as it stands; only the loop over independent
    signals is spread over the host's cores), in direct_form.decompose_batch's layout."""
    import concurrent.futures as cf
    import multiprocessing as mp

    S = np.atleast_2d(np.asarray(signals_, dtype=np.float64))
    B, n = S.shape
    max_imfs = kw.get("max_imfs", 10)
    workers = max(1, min(B, os.cpu_count() or 1, 16))
    # one BLAS / OpenMP thread per worker (the workers inherit the environment at spawn): B processes of
    # all-core BLAS pools would oversubscribe the host by a factor of its core count
    keep = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    os.environ.update(OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    try:
        with cf.ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as ex:
            res = list(ex.map(_one, [(S[b], kw) for b in range(B)]))
    finally:
        for k, v in keep.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    out = {"imfs": np.zeros((B, max_imfs + 1, n)), "count": np.zeros(B, np.int32),
           "l": np.zeros((B, max_imfs), np.int32), "N": np.zeros((B, max_imfs), np.int32),
           "margins": np.full((B, max_imfs + 1, 2), np.nan)}
    for b, d in enumerate(res):
        M = d["M"]
        out["imfs"][b] = d["imfs"]
        out["count"][b] = M
        out["l"][b, :M] = d["l"]
        out["N"][b, :M] = d["N"]
        out["margins"][b] = d["margins"]
    return out
