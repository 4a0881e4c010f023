#!/bin/bash
# K2 shape sweep (UNIAP_K2_V: buckets per thread at B = 1024)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=10 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for VV in 2 4; do
  for W in llama swin t5 bert vit; do
    UNIAP_K2_V=$VV timeout 600 python bench.py --steps 10 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/sweep_${W}_v$VV.json 2> gpurun_out/sweep_${W}_v$VV.err
  done
done
