"""Instruction mix of an ncu sass csv (dev tool): python tools/opmix.py <sass.csv> <signals*imfs*n>"""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; iS = h.index("Source"); iE = h.index("Instructions Executed")
op = Counter(); tot = 0
for r in rows[2:]:
    if len(r) < len(h): continue
    src = r[iS].split()
    if not src: continue
    m = src[1] if src[0].startswith('@') else src[0]
    e = int(r[iE] or 0); op[m.split('.')[0]] += e; tot += e
units = float(sys.argv[2])
fp64 = sum(op[k] for k in ['DMUL', 'DADD', 'DFMA', 'DSETP', 'DMNMX'])
print(f"total {tot}  per unit: all {tot*32/units:.1f}  fp64 {fp64*32/units:.1f}")
for k, v in op.most_common(22): print(f"  {k:8s} {v*32/units:7.2f}  {v/tot*100:5.1f}%")
