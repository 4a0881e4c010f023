"""bench.py -- the driver's benchmark contract for the exact UniAP strategy search.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]
    torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1, NCCL)

A "step" is one pass of the whole hot path (all rows) over
the synthetic profile of the workload: K1 cost tables -> K2 interval chain DP
-> K3/K4 stage combine (Eq. 2) -> K5 argmin + traceback -> record, and for
N > 1 the record exchange (NCCL all_gather over NVLink).  Candidate configs
are LPT-sharded across ranks (strong scaling: the search is fixed, more GPUs
finish it sooner).

value = DP cell-updates/s over all ranks with the profile resident in HBM
(device time by CUDA events on the launching stream, max over ranks);
e2e   = the same metric through the C ABI with HOST inputs: every step
        uploads the profile (H2D), runs, exchanges, and reads the result back.
Rank 0 prints ONE JSON line.  --impl reference times the CPU oracle
(oracle/, the reference arm of this tier) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "strategy-optimisation time (s) and DP cell-updates/s, 1/2/4/8 B200, vs CPU oracle"
UNIT = "cell-updates/s"
SM_COUNT = 148
ALU_LANES_PER_SM = 64  # 4 SMSPs x 16 lanes (alu pipe rt = 2 cycles per warp instruction, B300_MICROARCH.md)

WORKLOAD_NAMES = {"llama": "llama-7b-like", "bert": "bert-huge-like", "t5": "t5-large-like",
                  "vit": "vit-huge-like", "swin": "swin-huge-like"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(profile, cells, n_threads=None):
    """The oracle as it stands (oracle/, C, -O2 -march=native) on the host
    cores: the whole workload once on every core (threads over the candidate
    configs), and once on one thread (a bounded sample: ~1-20 s)."""
    from oracle import oracle
    oracle.build_oracle()
    n = n_threads or os.cpu_count() or 1
    t0 = time.perf_counter()
    res, _ = oracle.plan(profile, n_threads=n)
    dt = time.perf_counter() - t0
    t0 = time.perf_counter()
    res1, _ = oracle.plan(profile, n_threads=1)
    dt1 = time.perf_counter() - t0
    assert res1["objective"] == res["objective"]
    return {"value": cells / dt, "unit": UNIT, "cores": min(n, len(res["cfg_objective"])), "kind": "oracle",
            "sample": f"whole workload, 1 oracle run on {min(n, len(res['cfg_objective']))} threads ({dt:.2f} s) "
                      f"and 1 on one thread ({dt1:.2f} s); cells = the GPU path's canonical cells of the same workload",
            "seconds": dt, "single_thread": {"value": cells / dt1, "seconds": dt1, "cores": 1},
            "cpu_model": cpu_model(), "host_cores": os.cpu_count(), "objective": res["objective"]}


def bench_config(args, profile, ws, n_cfg):
    """The workload description both arms print (identical dicts)."""
    return {"workload": WORKLOAD_NAMES.get(args.workload, args.workload), "L": profile["model"]["L"],
            "devices_planned": profile["cluster"]["n_dev"], "B": profile["options"]["B"],
            "Q": profile["options"]["Q"], "candidates": n_cfg,
            "l2": "256 MiB memset between timed steps (flush)", "parallelism": f"configs-lpt{ws}"}


def measured_alu():
    """MEASURED_ALU.json (tools/alu_peak.py, this pool's B200): the DPX rate."""
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_ALU.json")))
    except (OSError, ValueError):
        return None


def run_reference(args, profile, cells):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import oracle
    oracle.build_oracle()
    n = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.plan(profile, n_threads=n)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res, _ = oracle.plan(profile, n_threads=n)
        times.append(time.perf_counter() - t0)
    ms = 1000 * statistics.mean(times)
    v = cells / (ms / 1000)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": bench_config(args, profile, ws, len(res["cfg_objective"])),
            "opt_time_s": ms / 1000.0,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": min(n, len(res["cfg_objective"])), "kind": "oracle",
                             "sample": f"whole workload per step, {args.steps} steps on {n} host threads",
                             "cpu_model": cpu_model(), "host_cores": os.cpu_count()},
            "objective": res["objective"]}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="llama", choices=sorted(WORKLOAD_NAMES))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from gen import profiles
    profile = profiles.make_profile(args.workload)

    import torch
    ws, rank, local = _dist()
    if args.impl == "reference":
        # the canonical cell count of the workload (the same unit as our arm),
        # counted on the host: the reference arm loads nothing of the product
        run_reference(args, profile, _cells_host(profile))
        return

    import torch.distributed as dist
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2307_16375_b200 as pkg

    # a dedicated (non-default) stream shared by the library, the timing
    # events and the NCCL exchange, so everything is ordered on one stream
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    h = pkg.Handle(local, stream.cuda_stream)
    RB = pkg.RECORD_BYTES
    rec = torch.zeros(RB, dtype=torch.uint8, device="cuda")
    all_recs = torch.zeros(ws * RB, dtype=torch.uint8, device="cuda")
    hdrs = torch.zeros(ws * RB, dtype=torch.uint8, device="cuda")  # phase-1 records (uniap_run_phase)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    # ---------------- device-resident: profile uploaded once ----------------
    h.prepare(profile)

    def step():
        if ws > 1:  # split run: only the owner of the global winner runs a traceback
            h.run_phase(rank, ws, rec.data_ptr(), 1)
            dist.all_gather_into_tensor(hdrs, rec)
            h.run_phase(rank, ws, rec.data_ptr(), 2, hdrs.data_ptr())
            dist.all_gather_into_tensor(all_recs, rec)
        else:
            h.run(rank, ws, rec.data_ptr())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    first = h.fetch()
    launches_per_step = first["n_launches"] // (args.warmup) if first["n_launches"] else 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times, dp_ms = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            if ws > 1:
                dist.barrier()
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            dp_ms.append(h.fetch()["ms_gpu_dp"])
    r = h.fetch()
    if ws > 1:  # the winner of the whole job (the timed steps ran the exchange): pick over every rank's record
        _, won = pkg.pick(all_recs.cpu().numpy().tobytes(), ws)
        r.update({k: won[k] for k in ("objective", "deg", "c")})
    ms_local = statistics.mean(times)
    # the workload size: cells of the canonical plan (one forward sweep per
    # start layer); the solver executes fewer (suffix
    # sweeps), so value = canonical cells / time is the effective rate, and
    # the roofline uses the relaxations actually executed.
    cells_local, relax_local = r["dp_cells_canonical"], r["dp_relax"]
    t = torch.tensor([ms_local, float(cells_local), float(relax_local)], dtype=torch.float64, device="cuda")
    if ws > 1:
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, cells = float(mx[0]), float(sm[1])
    else:
        ms, cells = ms_local, float(cells_local)
    value = cells / (ms / 1000.0)

    # ---------------- end to end through the C ABI, host inputs ------------
    # The profile is marshalled once into the ABI structs (pkg.Profile: host
    # arrays, what a C caller holds); each timed step validates and uploads
    # them (uniap_prepare: H2D), runs, and reads the result back.  The
    # Python dict -> struct conversion is timed separately (marshal_us).
    t0 = time.perf_counter()
    prof = pkg.Profile(profile)
    marshal_us = []
    for _ in range(5):
        t0 = time.perf_counter()
        pkg.Profile(profile)
        marshal_us.append((time.perf_counter() - t0) * 1e6)
    h.prepare(prof)  # resets the byte counters
    e2e_times = []
    e2e_steps = max(3, min(args.steps, 10))
    for i in range(e2e_steps + 1):
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if ws > 1:
            h.prepare(prof)                     # validation + H2D of the profile
            step()
            host = all_recs.cpu().numpy().tobytes()   # D2H of every rank's record
            st, res = pkg.pick(host, ws)
        else:
            res = h.plan(prof)                  # uniap_plan: prepare (H2D) + run + fetch (D2H)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i > 0:
            e2e_times.append(dt)
    counters = h.fetch()
    e2e_t = torch.tensor([statistics.mean(e2e_times)], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_t[0])
    h2d_per_step = counters["h2d_bytes"]
    d2h_per_step = counters["d2h_bytes"] + (ws * RB if ws > 1 else 0)

    if rank == 0:
        clocks = clk.summary()
        sm_max = clocks.get("sm_max_mhz") or 1965.0
        alu = measured_alu()
        if alu:
            peak = alu["peak_relax_per_s"] / 1e12  # T relax/s, measured (tools/alu_peak.py)
            peak_source = (f"measured: MEASURED_ALU.json (tools/alu_peak.py, {alu['when']}): "
                           f"{alu['viaddmnmx_per_clk_per_sm']:.1f} VIADDMNMX/clk/SM x {alu['sms']} SMs at "
                           f"{alu['clocks']['sm_mhz_median_under_load']} MHz under load")
        else:
            peak = SM_COUNT * ALU_LANES_PER_SM * sm_max * 1e6 / 1e12
            peak_source = (f"derived (MEASURED_ALU.json absent): {SM_COUNT} SMs x {ALU_LANES_PER_SM} alu lanes/clk x "
                           f"{sm_max:.0f} MHz (B300_MICROARCH alu pipe rt=2; DESIGN.md Sec. 4)")
        achieved = relax_local / (statistics.mean(dp_ms) / 1000.0) / 1e12 if dp_ms and dp_ms[0] > 0 else None
        traffic = None  # DRAM bytes of one step's forward K2 launches (ncu --set full, profiles/r2)
        summ = os.path.join(ROOT, "profiles", "r2", f"ncu_summary_{args.workload}.json")
        if os.path.exists(summ):
            try:
                traffic = json.load(open(summ)).get(f"dram_bytes_forward_step_{args.workload}")
            except Exception:
                traffic = None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": bench_config(args, profile, ws, len(r["cfg_objective"])),
            "opt_time_s": ms / 1000.0, "e2e_opt_time_s": e2e_s,
            "cells_executed_per_step": r["dp_cells"], "cells_canonical_per_step": r["dp_cells_canonical"],
            "cells_executed_per_s": float(r["dp_cells"]) * ws / (ms / 1000.0) if ws == 1 else None,
            "value_note": "value = canonical cells (one forward sweep per start layer: the problem size) / device "
                          "time, an effective rate; cells_executed_per_s = the cells the solver's plan executes",
            "e2e": {"value": cells / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d_per_step,
                    "d2h_bytes_per_step": d2h_per_step, "seconds_per_step": e2e_s,
                    "path": "uniap_plan = uniap_prepare (validate + H2D of the ABI profile) + uniap_run + uniap_fetch "
                            "(D2H + sync); N > 1: the split run (uniap_run_phase 1, NCCL all_gather of the headers, "
                            "phase 2, all_gather of the records) and uniap_pick",
                    "python_marshal_us": statistics.median(marshal_us)},
            "gpu_launches": launches_per_step,
            "roofline": {"bound": "alu", "kernel": "k2_chain (VIADDMNMX min-plus)", "achieved": achieved,
                         "peak": peak, "unit": "Trelax/s", "frac": (achieved / peak) if achieved else None,
                         "traffic": traffic,
                         "peak_source": peak_source,
                         "algorithmic_relax_per_step": relax_local, "k2_ms_per_step": statistics.mean(dp_ms),
                         "traffic_unit": "DRAM bytes read + written by one step's forward K2 launches (ncu --set "
                                         "full, cold cache: an upper bound; the tables + P a step needs are < 1 MB)"},
            "clocks": clocks,
            "objective": r["objective"], "plan": {"deg": r["deg"], "c": r["c"]},
        }
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(profile, cells)
        print(json.dumps(line), flush=True)
    h.close()
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def _cells_host(profile):
    """Algorithmic chain-DP cells of the workload without a GPU: a host mirror
    of the instance plan (only used by --impl reference on a GPU-less box)."""
    from oracle import oracle
    t, _, _ = oracle.build_tables(profile)
    L, Q, s = t["L"], t["cap"] + 1, t["skip_src"]
    cells = 0
    for cfg in t["cfgs"]:
        deg, S = cfg["deg"], cfg["n_strat"]
        if deg > L:
            continue
        for a in range(L):
            if deg == 1 and a > 0:
                break
            bmax = L - 1 if deg == 1 else L - 1 - deg + min(a + 1, deg)
            if bmax < a:
                continue
            n = bmax - a + 1
            copies = S if (s >= 0 and a <= s and bmax >= s + 2) else 1
            cells += copies * n * S * Q
    return cells


if __name__ == "__main__":
    main()
