#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=10 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/k2_latency.py > gpurun_out/lat_base.jsonl 2>&1
for W in llama t5 swin vit bert; do
  timeout 600 python bench.py --steps 10 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
done
