"""Writes tests/golden/cfg3_df_2p26.npz: the ORACLE's decomposition of the config-3 signal at its full size
(n = 2^26, BASELINE.json configs[3]) -- the expected values of tests/test_gpu_fullsize.py::test_cfg3_vs_direct_form.

Calls only oracle/ (oracle/direct_form.py, the paper's FFT direct form step by step, pinned to
the time-domain oracle in tests/test_oracle_pins.py) and the seeded input generator; nothing comes from the CUDA
path.  The full IMFs (11 x 512 MB) cannot be stored, so the file keeps what the GPU test compares:
  * the integers: M, l_m, N_m, the extrema counts k_m, and the oracle's decision margins (reading A21);
  * per slot (IMFs, trend): the 2-norm and the values at SAMPLE_IDX (4096 fixed indices spread over the signal,
    plus the first and last 64 samples, where the periodic wrap and the block boundaries of a distributed plan are).
The literal iteration (fif_oracle.c) cannot finish n = 2^26 (SURVEY.md hard part (iv)); the direct form is the
oracle used at this size.  Run once on a CPU box:  python tests/golden/make_cfg3_golden.py   (~10 min, ~12 GB)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import direct_form as df  # noqa: E402
from paper_1802_01359_b200 import signals  # noqa: E402

N_LOG2 = 26
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg3_df_2p26.npz")


def sample_idx(n: int) -> np.ndarray:
    step = n // 4096
    mid = np.arange(4096, dtype=np.int64) * step + (np.arange(4096, dtype=np.int64) * 7919) % step
    return np.unique(np.concatenate([np.arange(64), mid, np.arange(n - 64, n)]))


def main():
    n = 1 << N_LOG2
    s = signals.cfg3_signal(0, n=n)
    t0 = time.time()
    d = df.decompose(s, delta=signals.CONFIGS["cfg3"]["delta"])
    el = time.time() - t0
    M = d["M"]
    idx = sample_idx(n)
    norms = np.array([np.linalg.norm(d["imfs"][m]) for m in range(d["imfs"].shape[0])])
    samples = d["imfs"][:, idx].copy()
    np.savez_compressed(OUT, n=n, M=M, l=np.array(d["l"], np.int32), N=np.array(d["N"], np.int32),
                        k=np.array(d["k"], np.int64), margins=d["margins"], norms=norms, idx=idx, samples=samples,
                        snorm=np.linalg.norm(s), seconds=el)
    print(f"M={M} l={d['l']} N={d['N']} k={d['k']} ({el:.0f} s) -> {OUT}")


if __name__ == "__main__":
    main()
