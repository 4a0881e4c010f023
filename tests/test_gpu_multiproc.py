"""The multi-GPU product call through the real library: world 2 and 4
processes, each running its LPT share of the candidates with uniap_run on
cuda:0 (the round-end box has one GPU, so every rank shares it; gloo
carries the record exchange), Handle.plan_distributed's all_gather + pick --
the answer must equal the ORACLE's plan (objective, deg, c, stage_of,
strategy_of, costs, memory) on every rank (determinism across
world sizes)."""
import json
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

KEYS = ("objective", "deg", "c", "cfg_index", "stage_of", "strategy_of", "stage_cost", "cut_cost", "stage_mem")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, names, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2307_16375_b200 as pkg
    from gen import profiles
    h = pkg.Handle(0)
    out = {}
    for name in names:
        r = h.plan_distributed(profiles.make_profile(name))
        out[name] = {k: r[k] for k in KEYS + ("dp_relax",)}
    h.close()
    with open(os.path.join(outdir, f"r{rank}.json"), "w") as f:
        json.dump(out, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_plan_distributed_matches_oracle(orc, tmp_path, world):
    names = ["vit", "t5", "llama"]
    mp.spawn(_worker, args=(world, _free_port(), names, str(tmp_path)), nprocs=world, join=True)
    got = [json.load(open(tmp_path / f"r{r}.json")) for r in range(world)]
    for name in names:
        from gen import profiles
        want, _ = orc.plan(profiles.make_profile(name), n_threads=0)
        for r in range(world):
            for k in KEYS:
                assert got[r][name][k] == want[k], (world, r, name, k)
        assert all(got[r][name]["dp_relax"] == got[0][name]["dp_relax"] for r in range(world))
