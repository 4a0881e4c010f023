#!/bin/bash
# A/B: alternate two environment settings, 3 rounds, every workload (bench --no-cpu-baseline)
# usage: A="ENV=.." B="ENV=.." bash tools/ab.sh
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for R in 1 2 3; do
  for V in A B; do
    for W in ${WORKLOADS:-llama t5 swin vit bert}; do
      if [ $V = A ]; then E="$A"; else E="$B"; fi
      env $E timeout 300 python bench.py --steps 20 --warmup 3 --workload $W --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(json.dumps({'v':'$V','w':'$W','r':$R,'ms':d['ms_per_step'],'k2':d['roofline']['k2_ms_per_step']}))" >> gpurun_out/ab.jsonl
    done
  done
done
