#!/bin/bash
OUT=gpurun_out/r2h; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/hbm_probe tools/hbm_probe.cu && PROBE_ONLY=1 timeout 600 /tmp/hbm_probe > $OUT/hbm_probe2.jsonl 2> $OUT/hbm_probe2.err; echo "probe rc=$?"; cat $OUT/hbm_probe2.jsonl
