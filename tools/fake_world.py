"""Per-rank device time of the LPT shard plan at world 1/2/4/8, measured on
one GPU ("fake world": every rank's share runs alone, one after another),
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
        per = []
        for rank in range(world):
            for _ in range(3):
                h.run(rank, world, rec.data_ptr())
            torch.cuda.synchronize()
            ts = []
            for _ in range(10):
                h.run(rank, world, rec.data_ptr())
                ts.append(h.fetch()["ms_gpu_total"])
            per.append(statistics.median(ts))
        row[world] = {"ms_per_rank": [round(x, 4) for x in per], "max_ms": round(max(per), 4),
                      "balance": round(statistics.mean(per) / max(per), 3)}
    out[w] = row
    print(w, {k: (v["max_ms"], v["balance"]) for k, v in row.items()}, flush=True)
h.close()
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
