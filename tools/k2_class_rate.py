"""Per-class DPX efficiency of the forward K2 launches of one bench workload
step (UNIAP_TRACE diagnostics).

usage: python tools/k2_class_rate.py WORKLOAD [WORKLOAD ...]
For every forward K2 class: CTAs, summed CTA time, the relaxations its CTAs
executed ((n - 1) * S^2 * buckets of the CTA, from the per-CTA record of the
layer count n) and their rate per SM-us against the DPX peak of one SM
(MEASURED_ALU.json: VIADDMNMX per clock per SM x the SM clock).  Classes whose
CTAs share an SM (T < 512 without a cluster) count CTA time, not SM time, so
their efficiency reads low by the residency.
"""
import collections
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = os.path.join(tempfile.mkdtemp(), "trace.txt")
os.environ["UNIAP_TRACE"] = path
import torch  # noqa: E402
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import profiles  # noqa: E402

alu = json.load(open(os.path.join(ROOT, "MEASURED_ALU.json")))
rho = alu["viaddmnmx_per_clk_per_sm"]
mhz = alu["clocks"]["sm_mhz_median_under_load"]
per_sm_us = rho * mhz  # relaxations per SM-us at peak


def shape(tag):
    return dict(NS=tag & 63, V=(tag >> 6) & 15, T=((tag >> 10) & 63) * 32, C=(tag >> 16) & 31,
                DB=(tag >> 24) & 1, bw=(tag >> 25) & 1)


for w in sys.argv[1:] or ["llama"]:
    p = profiles.make_profile(w)
    h = pkg.Handle(0)
    h.prepare(p)
    for _ in range(5):
        h.run()
    torch.cuda.synchronize()
    open(path, "w").close()
    h.run()
    r = h.fetch()
    Q = p["options"]["Q"] if "options" in p else None
    recs = [tuple(int(x) for x in ln.split()) for ln in open(path).read().split("\n")[1:] if ln.strip()]
    by = collections.defaultdict(list)
    for tag, t0, t1, packed in recs:
        if tag >> 31:
            continue
        s = shape(tag)
        if s["bw"]:
            continue
        by[tag].append(((t1 - t0) / 1e3, (packed >> 40) & 0xFFFFFF))
    tot_r = tot_t = 0.0
    print(f"== {w}: step {r['ms_gpu_total']:.4f} ms, forward phase {r['ms_gpu_dp']:.4f} ms, "
          f"relax executed {r['dp_relax']:.3e}")
    for tag, v in sorted(by.items(), key=lambda kv: -sum(x[0] for x in kv[1])):
        s = shape(tag)
        q = Q or 1024
        bcta = min(s["T"] * s["V"], q)
        relax = sum(max(n - 1, 0) * s["NS"] ** 2 * bcta for _, n in v)
        sm_us = sum(d for d, _ in v)
        tot_r += relax
        tot_t += sm_us
        print(f"  NS{s['NS']:<2} V{s['V']} T{s['T']:<3} C{s['C']:<2} DB{s['DB']}  ctas {len(v):4d}  cta-us {sm_us:8.1f}  "
              f"relax {relax:.3e}  eff {relax / (sm_us * per_sm_us):.3f}")
    print(f"  all forward classes: eff {tot_r / (tot_t * per_sm_us):.3f} (relax from records {tot_r:.3e})")
    h.close()
