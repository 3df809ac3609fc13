"""Where a kernel spills: STL/LDL instructions of one function of a cubin, by innermost source line.
usage: python tools/spills.py <cubin> <mangled-name substring> [source file]   (dev tool)"""
import re
import subprocess
import sys
from collections import Counter

cubin, pat = sys.argv[1], sys.argv[2]
src_path = sys.argv[3] if len(sys.argv) > 3 else "/root/repo/paper_1802_01359_b200/csrc/fif_resident.cuh"
out = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout.split("\n")
inside, line, prev = False, None, False
cnt = Counter()
for ln in out:
    if re.match(r"\s*\.text\.", ln) or re.match(r"\s*\.section\s+\.text\.", ln):
        inside = pat in ln
        continue
    if not inside:
        continue
    m = re.search(r"line (\d+)", ln)
    if ln.strip().startswith("//##") and m:
        if not prev:
            line = int(m.group(1))
        prev = True
        continue
    prev = False
    for op in ("STL", "LDL"):
        if re.search(r"\b%s(\.\w+)*\b" % op, ln) and "/*" in ln:
            cnt[(line, op)] += 1
src = open(src_path).read().split("\n")
for (l, op), n in sorted(cnt.items(), key=lambda x: (x[0][0] or 0, x[0][1])):
    print(f"{l or 0:5} {op} {n:3}  {src[l - 1].strip()[:90] if l else ''}")
print("total", sum(cnt.values()))
