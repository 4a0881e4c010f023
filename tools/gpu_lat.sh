#!/bin/bash
mkdir -p gpurun_out
for F in 0 1; do UNIAP_K2_FLAGS=$F timeout 300 python tools/k2_latency.py > gpurun_out/lat_f$F.jsonl 2>&1; done
for CM in 0; do UNIAP_NO_GRAPH=1 timeout 300 python tools/k2_latency.py > gpurun_out/lat_nograph.jsonl 2>&1; done
