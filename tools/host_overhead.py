"""Host-side cost of each ABI call of one plan (GPU box): prepare / run / fetch,
wall-clock per call (after warm-up), and the whole uniap_plan."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import profiles  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "llama"
p = profiles.make_profile(w)
prof = pkg.Profile(p)
h = pkg.Handle(0)
for _ in range(5):
    h.plan(prof)
T = {"prepare": [], "run_launch": [], "wait_device": [], "fetch": [], "plan": []}
for _ in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); h.prepare(prof); t1 = time.perf_counter()
    h.run(); t2 = time.perf_counter()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    h.fetch(); t4 = time.perf_counter()
    T["prepare"].append(t1 - t0); T["run_launch"].append(t2 - t1); T["wait_device"].append(t3 - t2)
    T["fetch"].append(t4 - t3)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); h.plan(prof); T["plan"].append(time.perf_counter() - t0)
print(json.dumps({k: round(statistics.median(v) * 1e6, 1) for k, v in T.items()} | {"workload": w, "unit": "us"}))
