#!/bin/bash
# round-2 job T (1 GPU): the driver's view of this build: GPU suite, smoke,
# N=1 bench and reference arm at the defaults, launch list and one ncu
# --set full capture of the 256-bit commit kernel
OUT=gpurun_out/r2t; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:randomly > $OUT/pytest_gpu_1gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu_1gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "bench N=1 rc=$?"; cut -c1-300 $OUT/bench_n1.json
timeout 900 python bench.py --impl reference > $OUT/bench_ref_n1.json 2> $OUT/bench_ref_n1.err; echo "bench ref rc=$?"; cut -c1-200 $OUT/bench_ref_n1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 4 --warmup 3 --skip-cpu --e2e-steps 0 > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fold_direct_kernel -s 20 -c 1 -o $OUT/fold_direct_w256_full python bench.py --steps 4 --warmup 3 --skip-cpu --e2e-steps 0 > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"; ls -la $OUT/*.ncu-rep
