#!/bin/bash
mkdir -p gpurun_out
for V in ${VARIANTS:-base:variants/base new:.}; do
  name=${V%%:*}; dir=${V#*:}
  for W in ${WORKLOADS:-llama}; do
    (cd $dir && timeout 120 python tools/k2_trace.py $W) > gpurun_out/tr_${name}_$W.txt 2>&1
  done
done
