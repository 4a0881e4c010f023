"""K2 timeline of one bench workload step (UNIAP_TRACE diagnostics).

usage: python tools/k2_trace.py WORKLOAD [out.json]
Runs the workload's prepared plan a few times, then one traced run; prints per
kernel class: CTAs, first start / last end (us from the first K2 start), CTA
duration stats, and the SM occupancy (busy-SM count) over time.
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

w = sys.argv[1] if len(sys.argv) > 1 else "llama"
p = profiles.make_profile(w)
h = pkg.Handle(0)
h.prepare(p)
for _ in range(5):
    h.run()
torch.cuda.synchronize()
open(path, "w").close()
h.run()
h.fetch()
lines = open(path).read().split("\n")
recs = [tuple(int(x) for x in ln.split()) for ln in lines[1:] if ln.strip()]


KIND = {1: "K1 costs", 2: "K1d quantum", 3: "K1f quantise", 4: "fill", 5: "K4", 6: "K5a", 7: "K5c", 8: "K4 sorted", 9: "K4 loaded", 10: "K4 dp done", 11: "K5a winner", 12: "K5a stars", 13: "K5a ends", 14: "K4 H", 15: "K4 ends"}


def shape(tag):
    return dict(NS=tag & 63, V=(tag >> 6) & 15, T=((tag >> 10) & 63) * 32, C=(tag >> 16) & 31, G=(tag >> 21) & 7,
                DB=(tag >> 24) & 1, bw=(tag >> 25) & 1, grp=(tag >> 26) & 31)


t00 = min(r[1] for r in recs if not r[0] >> 31)  # time 0 = first K2 CTA
by = collections.defaultdict(list)
for tag, t0, t1, packed in recs:
    by[tag].append(((t0 - t00) / 1e3, (t1 - t00) / 1e3, packed & 255, (packed >> 40) & 0xFFFFFF))
out = []
for tag, v in sorted(by.items(), key=lambda kv: min(x[0] for x in kv[1])):
    s = shape(tag)
    d = sorted(x[1] - x[0] for x in v)
    if tag >> 31:
        name = KIND.get(tag & 255, "?") + (f" li0={(tag >> 8) & 0xFFFF}" if tag & 255 in (5, 8, 9, 10, 14, 15) else "")
    else:
        name = f"NS{s['NS']} V{s['V']} T{s['T']} C{s['C']} G{s['G']} DB{s['DB']}" + (" bw" if s["bw"] else "")
    row = dict(cls=name,
               ctas=len(v), start=round(min(x[0] for x in v), 1), end=round(max(x[1] for x in v), 1),
               dur_max=round(d[-1], 1), dur_med=round(d[len(d) // 2], 1), sm_us=round(sum(d), 1),
               us_per_layer=round(max((x[1] - x[0]) / max(x[3] - 1, 1) for x in v), 2))
    out.append(row)
    print(row)
    if os.environ.get("K2_TRACE_TOP") and not tag >> 31:  # the longest CTAs: (n layers, us)
        top = sorted(v, key=lambda x: x[0] - x[1])[:8]
        print("   longest (n, us, start):", [(x[3], round(x[1] - x[0], 1), round(x[0], 1)) for x in top])
# SM occupancy over time (10 us bins)
end = max(r[2] for r in recs)
nb = int((end - t00) / 1e4) + 1
busy = [set() for _ in range(nb)]
for tag, t0, t1, packed in recs:
    if t0 < t00:
        continue
    for b in range(int((t0 - t00) / 1e4), int((t1 - t00) / 1e4) + 1):
        busy[b].add(packed & 255)
occ = [len(b) for b in busy]
total = sum(x[1] - x[0] for tag, v in by.items() for x in v if not tag >> 31)
print("busy SMs per 10us:", occ)
print(f"span {(end - t00) / 1e3:.1f} us, CTA-us {total:.0f}, CTA-us / 148 = {total / 148:.1f} us")
if len(sys.argv) > 2:
    json.dump(dict(workload=w, classes=out, occupancy_10us=occ, span_us=(end - t00) / 1e3,
                   cta_us=total, records=recs), open(sys.argv[2], "w"))
