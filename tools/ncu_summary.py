"""Summarise ncu --set full reports of one bench step into profiles/<round>/.

usage: python tools/ncu_summary.py OUT.json WORKLOAD K2_REPORT [REST_REPORT]
K2_REPORT: the capture of one step's forward k2_chain launches only
(tools/profile_r2.sh); REST_REPORT: its K1 / K4 / K5 kernels.
"""
import csv
import io
import json
import subprocess
import sys

out, workload, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
rep = reps[0]


def load(r):
    raw = subprocess.run(["ncu", "-i", r, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    return rows[0], rows[1], rows[2:]


hdr, units, data = load(rep)
for r in reps[1:]:
    h2, u2, d2 = load(r)
    m = {h: i for i, h in enumerate(h2)}
    data += [[d[m[h]] if h in m else "" for h in hdr] for d in d2]
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
# the first report holds exactly one step's forward k2_chain launches
fwd = [k for k in kernels if "k2_chain" in k["kernel"]]
summ = {
    "workload": workload, "source": reps, "note": "ncu --set full --clock-control none, one bench step; times are "
    "serialized and cold-cache (compare shares, not absolutes)",
    "forward_k2_launches": len(fwd),
    "forward_k2_us_serialized": sum(k["us"] for k in fwd),
    # one step's forward K2 launches together (the unit of bench.py's roofline.achieved)
    f"dram_bytes_forward_step_{workload}": sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in fwd),
    f"dram_bytes_per_forward_launch_{workload}": (sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in fwd)
                                                 / max(len(fwd), 1)),
    "kernels": kernels}
json.dump(summ, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in summ.items() if k != "kernels"}))
