"""Launch overhead around one plan (GPU box): events around (1) a captured
torch graph of one tiny kernel and (2) one uniap_run of the workload, recorded
exactly as bench.py records a step (e0, host launch, e1; synchronised on both
sides, no flush), medians over 200 steps."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import profiles  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "llama"
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
x = torch.zeros(1024, device="cuda")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    x.add_(1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, n=200):
    for _ in range(10):
        fn()
    out = []
    for _ in range(n):
        torch.cuda.synchronize()
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3)
    return round(statistics.median(out), 2)


res = {"tiny_graph_us": timed(g.replay)}
h = pkg.Handle(0, s.cuda_stream)
h.prepare(pkg.Profile(profiles.make_profile(w)))
res["plan_step_us"] = timed(h.run)
r = h.fetch()
res.update(gpu_dp_us=round(r["ms_gpu_dp"] * 1e3, 2), gpu_total_us=round(r["ms_gpu_total"] * 1e3, 2))
print(json.dumps(res | {"workload": w}))
