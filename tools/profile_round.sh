#!/bin/bash
# Round profiling artifacts for the bench workload (1 GPU):
#  - bench line, clocks
#  - ncu launch list of the bench command (every launch, device time; serialized, cold cache)
#  - ncu --set full of every forward K2 launch of one step (+ K4, K5a) for traffic / pipe / stall numbers
mkdir -p gpurun_out
W=${WORKLOAD:-llama}
timeout 600 python bench.py --steps 20 --warmup 3 --workload $W > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
  python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline > /dev/null 2>&1
# launches per step: 17-19; skip the warm-up steps (graph replays are profiled per kernel node)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k2_chain|k4_vals|k5a|k5c|k1_" -s 60 -c 24 \
  -o gpurun_out/prof_full_$W python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/ncu_full_$W.log 2>&1
