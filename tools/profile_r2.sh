#!/bin/bash
# Round-2 profiling artifacts for one workload (1 GPU):
#  - ncu launch list of the bench command (every launch; serialised, cold cache)
#  - ncu --set full of one step's kernels (K1, K1d, K1f, K2 forward + backward, K4, K5a, K5c)
mkdir -p gpurun_out
W=${WORKLOAD:-llama}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
  python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k2_chain|k4_vals|k5a|k5c|k1_|k1d|k1f" -s 80 -c 40 \
  -o gpurun_out/prof_full_$W python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/ncu_full_$W.log 2>&1
