"""Inclusive executed-instruction and stall-sample shares per device FUNCTION of one kernel (dev tool).
Each SASS instruction's inline chain (nvdisasm -gi) is mapped to the functions of the source file whose
line ranges contain a frame; an instruction counts once for every distinct function on its chain.
usage: python tools/sass_funcs.py <ncu-rep> <cubin> <mangled kernel substring> [source file] [top]"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep, cubin, kern = sys.argv[1:4]
srcf = sys.argv[4] if len(sys.argv) > 4 else "/root/repo/paper_1802_01359_b200/csrc/fif_resident.cuh"
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40

# function ranges of the source file
src = open(srcf).read().split("\n")
starts = []
for i, ln in enumerate(src, 1):
    m = re.match(r"\s*(?:template\s*<.*>\s*)?(?:__device__|__global__|__host__ __device__)[^(]*?\b(\w+)\s*\(", ln)
    if m and not ln.strip().endswith(";"):
        starts.append((i, m.group(1)))
starts.sort()


def func_of(line):
    name = None
    for s, nm in starts:
        if s <= line:
            name = nm
        else:
            break
    return name


# ncu per-address counts for the kernel
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
cnt, stall = {}, {}
REASONS = ["stall_long_sb", "stall_short_sb", "stall_wait", "stall_barrier", "stall_mio", "stall_math", "stall_lg",
           "L1 Wavefronts Shared Excessive", "L1 Wavefronts Shared"]
extra = {}
cur, h, base = None, None, None
for r in csv.reader(io.StringIO(raw)):
    if r and r[0] == "Kernel Name":
        cur = r[1]
        continue
    if r and "Address" in r and "Source" in r:
        h = r
        continue
    if h is None or cur is None or (base is None and cnt) :
        continue
    if len(r) < len(h):
        continue
    d = dict(zip(h, r))
    a = d["Address"]
    if not (a.startswith("0x") or a.isdigit()):
        continue
    a = int(a, 16) if a.startswith("0x") else int(a)
    if base is None:
        base = a
    cnt[a - base] = int(d.get("Instructions Executed") or 0)
    stall[a - base] = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    extra[a - base] = [float(d.get(k) or 0) for k in REASONS]
    if len(cnt) and False:
        break

# inline chains from the cubin
out = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout.split("\n")
inside, chain, pending = False, [], []
fc, fs = Counter(), Counter()
fx = {}
tot_c = tot_s = 0
for ln in out:
    if re.match(r"\s*\.(section\s+)?\.?text\.", ln):
        inside = kern in ln
        continue
    if not inside:
        continue
    if ln.strip().startswith("//##"):
        # only frames of the source file (CUDA headers' lines, e.g. the shuffle intrinsics, are dropped)
        ls = [int(l) for f, l in re.findall(r'"([^"]+)", line (\d+)', ln) if f.endswith(srcf.split("/")[-1])]
        if not pending:
            chain = []
        pending.append(ls)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m:
        if pending:
            chain = sorted({x for p in pending for x in p})
            pending = []
        a = int(m.group(1), 16)
        c, s = cnt.get(a, 0), stall.get(a, 0)
        tot_c += c
        tot_s += s
        ex = extra.get(a, [0] * len(REASONS))
        for f in {func_of(x) for x in chain}:
            fc[f] += c
            fs[f] += s
            fx[f] = [u + v for u, v in zip(fx.get(f, [0] * len(REASONS)), ex)]
print(f"total executed {tot_c}  stall samples {tot_s}   (stall columns: % of all samples; smem: excess/all wavefronts)")
print(f"{'function':28} {'inst':>6} {'stall':>6} " + " ".join(f"{r.replace('stall_', ''):>8}" for r in REASONS[:7]) + "  smem-excess")
for f, c in fc.most_common(top):
    x = fx.get(f, [0] * len(REASONS))
    print(f"{str(f):28} {c / max(tot_c, 1) * 100:5.1f}% {fs[f] / max(tot_s, 1) * 100:5.1f}% " +
          " ".join(f"{v / max(tot_s, 1) * 100:7.1f}%" for v in x[:7]) + f"  {x[7]:.0f}/{x[8]:.0f}")
