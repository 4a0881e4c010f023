#!/bin/bash
# K2 shape sweep: bench llama / swin / t5 under different per-CTA bucket caps
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=10 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for BM in 4096 1024 512; do
  for W in llama swin t5 bert; do
    UNIAP_K2_BMAX=$BM timeout 600 python bench.py --steps 10 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/sweep_${W}_$BM.json 2> gpurun_out/sweep_${W}_$BM.err
  done
done
