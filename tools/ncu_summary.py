"""Summarise an ncu report (full set) into a small JSON for profiles/ (dev tool).
usage: python tools/ncu_summary.py <report.ncu-rep> <out.json> [label]"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
label = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
keys = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "smem_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "warps_active_per_sm": "sm__warps_active.avg.per_cycle_active",
    "registers_per_thread": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_per_block": "launch__shared_mem_per_block",
    "fp64_inst": "smsp__inst_executed_pipe_fp64.sum",
    "inst_executed": "smsp__inst_executed.sum",
}
res = []
for r in rows[2:]:
    d = dict(zip(h, r))
    u = dict(zip(h, units))
    e = {"kernel": d.get("Kernel Name", "")[:120], "label": label}
    for k, m in keys.items():
        v = d.get(m)
        if v in (None, ""):
            continue
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        unit = u.get(m, "")
        if unit == "Mbyte": x *= 1e6
        elif unit == "Gbyte": x *= 1e9
        elif unit == "Kbyte": x *= 1e3
        elif unit in ("msecond", "ms") and k == "duration_us": x *= 1e3
        elif unit in ("nsecond", "ns") and k == "duration_us": x *= 1e-3
        e[k] = x
    if "dram_read_bytes" in e and "dram_write_bytes" in e:
        e["dram_bytes"] = e["dram_read_bytes"] + e["dram_write_bytes"]
    stalls = {n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v)
              for n, v in d.items() if n.startswith("smsp__average_warps_issue_stalled_")
              and n.endswith("_per_issue_active.ratio") and v not in ("", None)}
    e["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:6])
    res.append(e)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
