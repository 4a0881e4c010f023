#!/bin/bash
# Round-2 profiling artifacts for one workload (1 GPU):
#  - ncu launch list of the bench command (every launch; serialised, cold cache)
#  - ncu --set full (with source) of one step's forward K2 launches, and
#    --set full of its K1 / K4 / K5 kernels; the per-step counts come from
#    the launch list (forward K2 = the k2_chain launches before k5a_winner)
mkdir -p gpurun_out
W=${WORKLOAD:-llama}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
  python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline > /dev/null 2>&1
read NK2 NF NO <<< $(python - "$W" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/launches_{sys.argv[1]}.csv")) if len(r) > 5]
ki = rows[0].index("Kernel Name")
names = [r[ki] for r in rows[1:]]
starts = [i for i, n in enumerate(names) if n.startswith("uniap::k1_costs")]
step = names[starts[0]:starts[1]]
k2 = [n for n in step if "k2_chain" in n]
k5 = next(i for i, n in enumerate(step) if "k5a_winner" in n)
nf = sum(1 for n in step[:k5] if "k2_chain" in n)
rest = [n for n in step if any(x in n for x in ("k1_costs", "k1d", "k1f", "k4_vals", "k5a", "k5c"))]
print(len(k2), nf, len(rest))
PY
)
echo "per step: k2 $NK2 forward $NF rest $NO" > gpurun_out/prof_counts_$W.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k2_chain" -s $((3 * NK2)) -c $NF \
  -o gpurun_out/prof_k2_$W python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/ncu_k2_$W.log 2>&1
timeout 1500 ncu --set full --clock-control none -k regex:"k1_|k1d|k1f|k4_vals|k5a|k5c" -s $((3 * NO)) -c $NO \
  -o gpurun_out/prof_rest_$W python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/ncu_rest_$W.log 2>&1
