"""Writes tests/golden/cfg0_noise_free.json: the ORACLE's decomposition of noise-free config 0
(BASELINE.json configs[0] with sigma = 0: sin(2 pi 2x) + 0.5 sin(2 pi 16x) + 0.25 sin(2 pi 64x), n = 1024,
x_j = j/n; xi = 1.6, delta = 1e-3, max_inner = 200, max_imfs = 10), Algorithm 2 iterated
literally by oracle/fif_oracle.c.  Calls only oracle/ and the seeded generator.  The same integers were
computed independently by the survey's throwaway numpy model (SURVEY.md §8c "noise-free cfg0 fixture", E9);
tests/test_oracle_pins.py checks the two agree.  Run: python tests/golden/make_cfg0_golden.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1802_01359_b200 import signals  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg0_noise_free.json")


def main():
    s = signals.cfg0_signal(0, noise=0.0)[None, :]
    r = oracle.decompose(s)
    M = int(r["count"][0])
    mg = r["margins"][0]
    doc = {
        "cite": "PAPER.md:401-417 (Alg. 2), :431 (SD), :81 (l); oracle/fif_oracle.c via tests/golden/make_cfg0_golden.py",
        "signal": "cfg0 with sigma = 0 (signals.cfg0_signal(0, noise=0.0)), n = 1024",
        "params": {"xi": 1.6, "delta": 1e-3, "max_inner": 200, "max_imfs": 10, "window": "tri_sq (R1)"},
        "M": M,
        "k": [int(x) for x in r["k"][0][:M + 1]],
        "l": [int(x) for x in r["l"][0][:M]],
        "N": [int(x) for x in r["N"][0][:M]],
        "imf_norm_over_s_norm": [float(x) for x in
                                 (np.linalg.norm(r["imfs"][0], axis=1) / np.linalg.norm(s[0]))[:M + 1]],
        "margins_extrema": [None if not np.isfinite(x) else float(x) for x in mg[:M + 1, 0]],
        "margins_sd": [None if not np.isfinite(x) else float(x) for x in mg[:M, 1]],
    }
    json.dump(doc, open(OUT, "w"), indent=1)
    print(json.dumps({k: doc[k] for k in ("M", "k", "l", "N")}))


if __name__ == "__main__":
    main()
