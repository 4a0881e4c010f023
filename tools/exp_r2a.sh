#!/bin/bash
# round-2 experiment: one bucket per thread for the deg = 1 chain clusters
mkdir -p gpurun_out
for W in llama t5; do
  timeout 120 python tools/k2_trace.py $W > gpurun_out/trace_base_$W.txt 2>&1
  UNIAP_K2_SV1=1 timeout 120 python tools/k2_trace.py $W > gpurun_out/trace_sv1_$W.txt 2>&1
done
NO_TESTS=1 VARIANTS="base:X=0 sv1:UNIAP_K2_SV1=1" bash tools/gpu_ab.sh > gpurun_out/ab_summary.txt 2>&1
