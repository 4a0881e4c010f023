"""Summarise an ncu --set full report of one bench step into profiles/<round>/.

usage: python tools/ncu_summary.py gpurun_out/prof_full_llama.ncu-rep profiles/r1/ncu_k2_summary.json llama
Forward K2 launches = the k2_chain launches between the first k1_costs and the next k5a_winner.
"""
import csv
import io
import json
import subprocess
import sys

rep, out, workload = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def f(d, k):
    try:
        return float(d[ix[k]])
    except (KeyError, ValueError):
        return None


def kb(d, k):  # ncu reports Kbyte / Mbyte / byte units per column
    u = units[ix[k]].lower()
    v = f(d, k) or 0.0
    return v * (1e3 if u.startswith("k") else 1e6 if u.startswith("m") else 1.0)


kernels = []
for d in data:
    name = d[ix["Kernel Name"]]
    stalls = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): f(d, h)
              for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")}
    top = sorted(((v, k) for k, v in stalls.items() if v), reverse=True)[:5]
    kernels.append({
        "kernel": name, "us": f(d, "gpu__time_duration.sum"), "grid": d[ix["launch__grid_size"]],
        "block": d[ix["launch__block_size"]], "regs": f(d, "launch__registers_per_thread"),
        "dram_read_bytes": kb(d, "dram__bytes_read.sum"), "dram_write_bytes": kb(d, "dram__bytes_write.sum"),
        "alu_pipe_active_pct": f(d, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": f(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": f(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "top_stalls": {k: round(v, 2) for v, k in top}})
# forward K2 of one step: k2 launches before the first k5a
fwd, seen_k1 = [], False
for k in kernels:
    if "k1_costs" in k["kernel"]:
        seen_k1 = True
    elif "k5a" in k["kernel"] and seen_k1:
        break
    elif "k2_chain" in k["kernel"] and seen_k1:
        fwd.append(k)
summ = {
    "workload": workload, "source": rep, "note": "ncu --set full --clock-control none, one bench step; times are "
    "serialized and cold-cache (compare shares, not absolutes)",
    "forward_k2_launches": len(fwd),
    "forward_k2_us_serialized": sum(k["us"] for k in fwd),
    f"dram_bytes_per_launch_{workload}": sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in fwd),
    "kernels": kernels}
json.dump(summ, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in summ.items() if k != "kernels"}))
