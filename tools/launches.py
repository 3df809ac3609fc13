"""Summarise an ncu --csv launch list: per kernel count, total/avg time, share, DRAM GB/s."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, collections.defaultdict(dict)
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = data[int(d["ID"])]
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
            e["name"] = d["Kernel Name"].split("(")[0].replace("void ", "")
            e["grid"] = d["Grid Size"]
    return data


def summary(path):
    data = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in data.values():
        a = agg[d["name"]]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:40s} n={a[0]:4d} t={a[1] / 1e3:9.1f}us avg={a[1] / a[0] / 1e3:8.1f}us {100 * a[1] / tot:5.1f}% "
                   f"dram={a[2] / max(a[1], 1):6.0f} GB/s")
    out.append(f"total {tot / 1e3:.1f} us over {len(data)} launches")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        print(summary(p))
