"""Small decompositions covering every regime, run under compute-sanitizer (one tool per gpurun call; dev tool):
config 0, a 64-signal config-1 batch (resident, per-L table on and off), one streamed mixed-radix plan,
an emulated 4-rank distributed plan (collective and peer mode), fp32 resident + streamed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1802_01359_b200 import fif, signals  # noqa: E402


def run(plan, s):
    x = torch.from_numpy(np.ascontiguousarray(s)).cuda()
    out = plan.alloc_outputs()
    plan.decompose(x, *out)
    torch.cuda.synchronize()
    return [t.cpu() for t in out]


torch.cuda.set_device(0)
B = int(os.environ.get("SAN_B", "64"))
run(fif.Plan(1024, 1, "f64"), signals.make_batch("cfg0"))
s1 = signals.make_batch("cfg1", batch=B)
run(fif.Plan(4096, B, "f64"), s1)
p = fif.Plan(4096, B, "f64")
p.set_eigen_table(True)
run(p, s1)
s3 = np.stack([signals.tones_signal(3 * 1024, 21, i) for i in range(3)])
run(fif.Plan(3 * 1024, 3, "f64", regime=fif.REGIME_STREAMED), s3)
run(fif.Plan(1 << 14, 2, "f32", regime=fif.REGIME_STREAMED), np.stack([signals.cfg4_signal(1 << 14, i) for i in range(2)]))
run(fif.Plan(1024, 8, "f32"), np.stack([signals.cfg4_signal(1024, i) for i in range(8)]))
full = signals.cfg3_signal(0, n=1 << 16)
run(fif.Plan.dist(1 << 16, 0, 4, emulated=True), full.reshape(4, -1))
os.environ["FIF_DIST_PEER"] = "1"
run(fif.Plan.dist(1 << 16, 0, 4, emulated=True), full.reshape(4, -1))
print("sanitize cases done")
