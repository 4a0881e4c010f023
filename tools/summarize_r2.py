"""Build profiles/r2/ from a tools/final_r2.sh session (gpurun_out/final):
copies the raw artifacts and writes SUMMARY.md's per-workload table and the
BASELINE.md §3 rows (printed)."""
import glob
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "final")
DST = os.path.join(ROOT, "profiles", "r2")
os.makedirs(os.path.join(DST, "sanitizer"), exist_ok=True)


def last_json(path):
    try:
        return json.loads(open(path).read().strip().splitlines()[-1])
    except Exception:
        return None


for f in glob.glob(os.path.join(SRC, "*")):
    b = os.path.basename(f)
    if os.path.isdir(f):
        continue
    if b.endswith((".json", ".txt", ".log", ".csv")):
        shutil.copy(f, os.path.join(DST, b))
for f in glob.glob(os.path.join(SRC, "san", "*.log")):
    shutil.copy(f, os.path.join(DST, "sanitizer", os.path.basename(f)))

rows = []
for w in ("llama", "t5", "swin", "vit", "bert"):
    d = last_json(os.path.join(SRC, f"bench_{w}.json"))
    if not d:
        continue
    rf, cb, e = d["roofline"], d.get("cpu_baseline", {}), d["e2e"]
    rows.append((w, d["config"]["candidates"], d["cells_canonical_per_step"], d["cells_executed_per_step"],
                 rf["algorithmic_relax_per_step"], d["ms_per_step"], rf["k2_ms_per_step"], d["value"],
                 d.get("cells_executed_per_s"), rf["achieved"], rf["frac"], 1e3 * e["seconds_per_step"],
                 cb.get("single_thread", {}).get("seconds"), cb.get("seconds"), cb.get("cpu_model"),
                 cb.get("cores"), d["plan"], d["objective"], d["clocks"]["sm_mhz"]))
hdr = ("| workload | #(deg,c) | cells (canonical) | cells executed | relaxations executed | step ms (device) | "
       "K2 fwd ms | cell-updates/s (canonical) | executed cells/s | T relax/s | frac of DPX peak | e2e ms | "
       "oracle s (1 thr) | oracle s (all thr) | plan (deg, c) | SM MHz |")
lines = [hdr, "|" + "---|" * 16]
for r in rows:
    lines.append(f"| {r[0]} | {r[1]} | {r[2]:.3g} | {r[3]:.3g} | {r[4]:.3g} | {r[5]:.4f} | {r[6]:.4f} | {r[7]:.3g} | "
                 f"{(r[8] or 0):.3g} | {r[9]:.2f} | {r[10]:.3f} | {r[11]:.3f} | {(r[12] or 0):.2f} | "
                 f"{(r[13] or 0):.2f} ({r[15]}) | {r[16]['deg']}, {r[16]['c']} | {r[18]} |")
table = "\n".join(lines)
print(table)
open(os.path.join(DST, "table.md"), "w").write(table + "\n")
if rows:
    print("CPU:", rows[0][14])
