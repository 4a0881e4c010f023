#!/bin/bash
# ncu --set full of the K2 launches of one llama step, schedule A vs B (env)
mkdir -p gpurun_out
for V in 0 1; do
  UNIAP_K2_SEG=$V timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_chain" -s 40 -c 14 \
    -o gpurun_out/prof_seg$V python bench.py --steps 2 --warmup 3 --workload ${WORKLOAD:-llama} --no-cpu-baseline > gpurun_out/ncu_seg$V.log 2>&1
done
