"""Opcode histogram of an ncu --page source --csv dump (SASS view): executed warp-instructions and
warp-stall samples per opcode.  python tools/sass_hist.py src.csv [topN]"""
import csv
import sys
from collections import Counter


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def hist(path, top=25):
    r = list(csv.reader(open(path)))
    h = r[1]
    rows = [x for x in r[2:] if len(x) == len(h)]
    iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    tot = sum(num(x[iW]) for x in rows) or 1
    totE = sum(num(x[iE]) for x in rows) or 1
    c, cs = Counter(), Counter()
    for x in rows:
        t = x[iS].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        op = op.split(".")[0]
        c[op] += num(x[iE])
        cs[op] += num(x[iW])
    print(f"warp-instructions {totE}, stall samples {tot}")
    for k, v in c.most_common(top):
        print(f"{k:10s} {v:12d} {100 * v / totE:5.1f}%  stall {100 * cs[k] / tot:5.1f}%")


if __name__ == "__main__":
    hist(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
