"""Per-rank device time of the LPT shard plan at world 1/2/4/8, measured on
one GPU ("fake world": every rank's share runs alone, one after another,
as the split run: phase 1, gathered headers, phase 2),
for each bench workload -> the predicted device time of a real N-GPU run
(the max over ranks) and its load balance.

usage: python tools/fake_world.py [out.json]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import profiles  # noqa: E402

out = {}
h = pkg.Handle(0)
rec = torch.zeros(pkg.RECORD_BYTES, dtype=torch.uint8, device="cuda")
for w in ("llama", "t5", "swin", "vit", "bert"):
    p = profiles.make_profile(w)
    h.prepare(p)
    row = {}
    for world in (1, 2, 4, 8):
        # the split run of bench.py / plan_distributed: phase 1 on every rank,
        # the headers gathered, phase 2 (the traceback only on the winner's
        # owner); a rank's device time = its phase 1 + its phase 2
        hdrs = torch.zeros(world * pkg.RECORD_BYTES, dtype=torch.uint8, device="cuda")
        recs = [torch.zeros(pkg.RECORD_BYTES, dtype=torch.uint8, device="cuda") for _ in range(world)]
        per = []
        t1 = {}
        for rank in range(world):
            if world == 1:
                continue
            ts = []
            for i in range(13):
                h.run_phase(rank, world, recs[rank].data_ptr(), 1)
                if i >= 3:
                    ts.append(h.fetch()["ms_gpu_total"])
            t1[rank] = statistics.median(ts)
            hdrs[rank * pkg.RECORD_BYTES:(rank + 1) * pkg.RECORD_BYTES].copy_(recs[rank])
        torch.cuda.synchronize()
        for rank in range(world):
            ts = []
            for i in range(13):
                if world == 1:
                    h.run(rank, world, rec.data_ptr())
                else:
                    h.run_phase(rank, world, recs[rank].data_ptr(), 1)
                    h.run_phase(rank, world, recs[rank].data_ptr(), 2, hdrs.data_ptr())
                if i >= 3:
                    ts.append(h.fetch()["ms_gpu_total"] + t1.get(rank, 0.0))
            per.append(statistics.median(ts))
        row[world] = {"ms_per_rank": [round(x, 4) for x in per], "max_ms": round(max(per), 4),
                      "balance": round(statistics.mean(per) / max(per), 3)}
    out[w] = row
    print(w, {k: (v["max_ms"], v["balance"]) for k, v in row.items()}, flush=True)
h.close()
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
