#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/k2_latency.py > gpurun_out/lat_base.jsonl 2>&1
# profile the first case's K2 launches (deg=1, S=21, Q=4096) and the S=10 Q=1024 chain
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_chain -s 2 -c 1 \
  -o gpurun_out/prof_lat21 python tools/k2_latency.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_chain -s 34 -c 1 \
  -o gpurun_out/prof_lat10 python tools/k2_latency.py > /dev/null 2>&1
