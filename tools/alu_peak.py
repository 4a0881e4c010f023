"""Measure the K2 roofline denominator (DPX VIADDMNMX rate) with the SM
clock sampled meanwhile, and write MEASURED_ALU.json at the repo root
(bench.py's roofline.peak reads it).

    python tools/alu_peak.py [seconds]
"""
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tools", "alu_peak.cu")
BIN = os.path.join(ROOT, "build", "alu_peak")


def main():
    secs = sys.argv[1] if len(sys.argv) > 1 else "2"
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", BIN, SRC],
                   check=True)
    q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    smi = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100", "-i",
                            "0"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    time.sleep(0.3)
    out = subprocess.run([BIN, secs], capture_output=True, text=True, check=True).stdout
    time.sleep(0.2)
    smi.terminate()
    rows = [r.split(", ") for r in smi.communicate()[0].strip().splitlines() if r.strip()]
    res = json.loads(out.strip().splitlines()[-1])
    sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
    busy = [x for x in sm if x > 500]
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 3 + i and r[3 + i].lower() == "active"})
    res.update({
        "what": "K2 roofline denominator: DPX VIADDMNMX (one min-plus relaxation) per second on the whole GPU",
        "peak_relax_per_s": res["relax_per_s_median"],
        "clocks": {"sm_mhz_median_under_load": statistics.median(busy) if busy else None,
                   "sm_max_mhz": max(float(r[1]) for r in rows) if rows else None, "samples": len(rows),
                   "reasons": reasons},
        "how": "tools/alu_peak.cu: 148 x 8 CTAs x 256 threads x 16 independent __viaddmin_s32 chains, repeated for "
               f"{secs} s; wall time per launch from %globaltimer (first CTA start to last CTA end), median over "
               "launches; per-SM rate from %clock64 (median over SMs); nvidia-smi sampled every 100 ms meanwhile",
        "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    })
    with open(os.path.join(ROOT, "MEASURED_ALU.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
