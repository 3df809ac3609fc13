"""Time fif_decompose on config 1 with an alternative build of the library (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1802_01359_b200 import fif, signals
eig = "--eig" in sys.argv
f32 = "--f32" in sys.argv
sys.argv = [a for a in sys.argv if a not in ("--eig", "--f32")]
if len(sys.argv) > 1:
    fif.LIB_PATH = os.path.abspath(sys.argv[1])
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
s = signals.make_batch("cfg4", batch=min(B, 4096), n=n) if f32 else signals.make_batch("cfg1", batch=B, n=n)
if B > s.shape[0]:
    s = np.concatenate([s] * ((B + s.shape[0] - 1) // s.shape[0]))[:B]
x = torch.from_numpy(np.ascontiguousarray(s)).cuda()
plan = fif.Plan(n, B, "f32" if f32 else "f64")
if eig:
    plan.set_eigen_table(True)
out = plan.alloc_outputs()
for _ in range(3): plan.decompose(x, *out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): plan.decompose(x, *out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"{sys.argv[1] if len(sys.argv)>1 else 'default'}: n={n} B={B} {ms:.3f} ms  {B*n/ms/1e6:.3f} Gsamples/s  launch={plan.launch_config()}  M={out[1].float().mean().item():.2f}")
