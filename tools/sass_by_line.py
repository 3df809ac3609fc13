"""Attribute ncu per-instruction stall samples / executed instructions of ONE kernel to source lines of
one file (the outermost inlined frame that lies inside [lo, hi] of that file).  Dev tool.
usage: sass_by_line.py <ncu-rep> <cubin> <mangled kernel name> <source file> <lo> <hi> [top] [inner|outer]"""
import csv, io, os, re, subprocess, sys
from collections import Counter

rep, cubin, kern, srcf, lo, hi = sys.argv[1:7]
lo, hi = int(lo), int(hi)
top = int(sys.argv[7]) if len(sys.argv) > 7 else 40
MODE = sys.argv[8] if len(sys.argv) > 8 else "outer"
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
# one block per kernel in the report: pick the one whose name contains $NCU_KSUB (default: the first)
ksub = os.environ.get("NCU_KSUB", "")
blocks, name, h = [], None, None
for r in csv.reader(io.StringIO(raw)):
    if r and r[0] == "Kernel Name":
        name = r[1]
        continue
    if r and "Address" in r and "Source" in r:
        h = r
        blocks.append((name, h, []))
        continue
    if blocks and len(r) == len(blocks[-1][1]):
        blocks[-1][2].append(r)
name, h, body = next(b for b in blocks if ksub in (b[0] or ""))
iA, iS, iW, iE = (h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed"))
data, base = [], None
for r in body:
    a = int(r[iA], 16) if r[iA].startswith("0x") else int(r[iA])
    base = a if base is None else base
    data.append((a - base, r[iS], int(r[iW] or 0), int(r[iE] or 0)))
sym = subprocess.run(["readelf", "-sW", cubin], capture_output=True, text=True).stdout
idx = next(l.split(":")[0].strip() for l in sym.splitlines() if l.rstrip().endswith(" " + kern) and "FUNC" in l)
lst = subprocess.run(["nvdisasm", "-gi", "-fun", idx, cubin], capture_output=True, text=True).stdout.splitlines()
amap, cur, chain, prevc, infunc = {}, None, [], False, False
for ln in lst:
    st = ln.strip()
    if st.startswith(".section") or st.startswith(".text."):
        infunc = (".text." + kern) in st
    if not infunc:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if st.startswith("//##") and m:
        if not prevc:
            chain = []
        chain.append((int(m.group(2)), m.group(1).split("/")[-1] == srcf.split("/")[-1]))
        prevc = True
        continue
    if prevc:
        ks = [l for l, f in chain if f and lo <= l <= hi]
        cur = (ks[0] if MODE == "inner" else ks[-1]) if ks else None
    prevc = False
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        amap[int(m.group(1), 16)] = cur
tot, totE = sum(d[2] for d in data), sum(d[3] for d in data)
bys, bye = Counter(), Counter()
for a, s, w, e in data:
    bys[amap.get(a)] += w
    bye[amap.get(a)] += e
src = open(srcf).read().split("\n")
for l, w in bys.most_common(top):
    print(f"{l} st {w / tot * 100:5.1f}% inst {bye[l] / totE * 100:5.1f}% | {src[l - 1].strip()[:90] if l else ''}")
