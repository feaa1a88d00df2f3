#!/bin/bash
# round-2 job G (1 GPU): guard-band out-of-bounds tests (compute-sanitizer is
# closed on this pool), the HBM ceiling probe, the N=1 bench.
OUT=gpurun_out/r2g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_guards.py -q -p no:randomly > $OUT/pytest_guards.log 2>&1; echo "guards rc=$?"; tail -5 $OUT/pytest_guards.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/hbm_probe tools/hbm_probe.cu && timeout 600 /tmp/hbm_probe > $OUT/hbm_probe.jsonl 2> $OUT/hbm_probe.err; echo "probe rc=$?"; cat $OUT/hbm_probe.jsonl
timeout 600 python bench.py --skip-cpu --e2e-steps 0 > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "bench N=1 rc=$?"; cut -c1-300 $OUT/bench_n1.json
