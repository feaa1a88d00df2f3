#!/bin/bash
# round-2 job AU (1 GPU): the driver's view of the current build: GPU suite,
# smoke, N=1 bench and reference arm at the defaults
OUT=gpurun_out/r2au; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > $OUT/pytest_gpu_1gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu_1gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "bench N=1 rc=$?"; cut -c1-300 $OUT/bench_n1.json
timeout 900 python bench.py --impl reference > $OUT/bench_ref_n1.json 2> $OUT/bench_ref_n1.err; echo "bench ref rc=$?"; cut -c1-200 $OUT/bench_ref_n1.json
