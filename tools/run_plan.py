"""Run fif_decompose on a synthetic config batch `reps` times (profiling driver: ncu / timing).
python tools/run_plan.py --config cfg2 [--batch B] [--n N] [--reps R] [--dtype f64]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1802_01359_b200 import fif, signals  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--regime", type=int, default=0)
ap.add_argument("--eig", action="store_true", help="per-L eigenvalue table (fif_plan_set_eigen_table)")
a = ap.parse_args()
if a.config == "cfg4":
    s = signals.make_batch("cfg4", batch=a.batch or 64, n=a.n)
    dtype, delta = "f32", 1e-3
else:
    c = signals.CONFIGS[a.config]
    B = a.batch or c["batch"]
    s = signals.make_batch(a.config, batch=min(B, 64), n=a.n)
    if B > s.shape[0]:
        s = np.concatenate([s] * ((B + s.shape[0] - 1) // s.shape[0]))[:B]
    dtype, delta = c["dtype"], c["delta"]
plan = fif.Plan(s.shape[1], s.shape[0], dtype, delta=delta, regime=a.regime)
if a.eig:
    plan.set_eigen_table(True)
x = torch.from_numpy(np.ascontiguousarray(s)).cuda()
out = plan.alloc_outputs()
for r in range(a.reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    plan.decompose(x, *out)
    torch.cuda.synchronize()
    print(f"rep {r}: {1e3 * (time.perf_counter() - t):.3f} ms  kernels/call {plan.launch_config()}", flush=True)
