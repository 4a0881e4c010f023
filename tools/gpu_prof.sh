#!/bin/bash
# profiling session: bench, launch list (ncu, serialized cold-cache) and a full ncu capture of K2
mkdir -p gpurun_out
W=${WORKLOAD:-llama}
timeout 600 python bench.py --steps 10 --warmup 3 --workload $W > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
  python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/ncu_launch_bench_$W.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k2_chain -s 6 -c 6 \
  -o gpurun_out/prof_k2_$W python bench.py --steps 1 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/ncu_full_$W.log 2>&1
ls -la gpurun_out
