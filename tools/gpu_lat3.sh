#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/lat3.jsonl; : > $o
timeout 120 python tools/k2_lat3.py base >> $o 2>&1
UNIAP_K2_FLAGS=1 timeout 120 python tools/k2_lat3.py relaxed >> $o 2>&1
UNIAP_K2_SINGLE=0 timeout 120 python tools/k2_lat3.py nosingle >> $o 2>&1
UNIAP_K2_BMAX=256 timeout 120 python tools/k2_lat3.py bmax256 >> $o 2>&1
UNIAP_K2_FLAGS=8 timeout 120 python tools/k2_lat3.py noG >> $o 2>&1
