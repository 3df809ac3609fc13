"""Attribute ncu per-SASS-address counts to source lines (innermost inlined line). Dev tool.
usage: sass_lines.py <ncu sass csv> <nvdisasm -gi kernel listing> [top]"""
import csv, re, sys
from collections import Counter, defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iA, iS, iW, iE = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
cnt, stall, ops = {}, {}, {}
base = None
for r in rows[2:]:
    if len(r) < len(h) or not (r[iA].startswith("0x") or r[iA].isdigit()): continue
    a = int(r[iA], 16) if r[iA].startswith("0x") else int(r[iA])
    if base is None: base = a
    a -= base
    cnt[a] = int(r[iE] or 0); stall[a] = int(r[iW] or 0); ops[a] = r[iS].split()[0] if r[iS] else ""
line = None
prev_comment = False
byline, byline_st, byline_ops = Counter(), Counter(), defaultdict(Counter)
for ln in open(sys.argv[2]):
    m = re.search(r'line (\d+)', ln)
    if ln.strip().startswith("//##") and m:
        if not prev_comment:
            line = int(m.group(1))  # innermost line of an inline chain comes first
        prev_comment = True
        continue
    prev_comment = False
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*)', ln)
    if m:
        a = int(m.group(1), 16)
        if a in cnt:
            byline[line] += cnt[a]; byline_st[line] += stall[a]
            op = m.group(2).split()[0]
            if op.startswith('@'): op = m.group(2).split()[1]
            byline_ops[line][op.split('.')[0]] += cnt[a]
tot = sum(byline.values()); tst = sum(byline_st.values())
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
src = open(sys.argv[4] if len(sys.argv) > 4 else "/root/repo/paper_1802_01359_b200/csrc/fif_resident.cuh").read().split("\n")
for l, c in byline.most_common(top):
    s = src[l - 1].strip()[:70] if l else ""
    print(f"{l or 0:5} {c/tot*100:5.1f}% st {byline_st[l]/tst*100:5.1f}%  {dict(byline_ops[l].most_common(4))}  | {s}")
