#!/bin/bash
# round-2 job E (1 GPU): compute-sanitizer (memcheck, racecheck, synccheck,
# initcheck) over the single-GPU parity tests, smoke, the N=1 bench, its
# launch list and one ncu --set full capture of the dominant kernel.
OUT=gpurun_out/r2e; mkdir -p $OUT
nvidia-smi -L > $OUT/gpus.txt
CS=compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 99 python -m pytest -q -p no:randomly tests/test_gpu_fold.py tests/test_gpu_kacc.py tests/test_gpu_commit.py -k "not full_size and not multidevice" > $OUT/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 $OUT/memcheck.log
timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 99 python -m pytest -q -p no:randomly tests/test_gpu_protocol.py -x > $OUT/memcheck_protocol.log 2>&1; echo "memcheck protocol rc=$?"; tail -4 $OUT/memcheck_protocol.log
timeout 1200 $CS --tool racecheck --racecheck-report hazard --error-exitcode 99 python -m pytest -q -p no:randomly tests/test_gpu_fold.py -k "tree_commit_matches_oracle or fold_variants_agree or random_stack or bf16_leaves or fixed_programs" > $OUT/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -4 $OUT/racecheck.log
timeout 1200 $CS --tool synccheck --error-exitcode 99 python -m pytest -q -p no:randomly tests/test_gpu_fold.py tests/test_gpu_kacc.py -k "not full_size and not multidevice" > $OUT/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -4 $OUT/synccheck.log
timeout 900 $CS --tool initcheck --error-exitcode 99 python -m pytest -q -p no:randomly tests/test_gpu_fold.py -k "tree_commit_matches_oracle or fold_variants_agree or golden" > $OUT/initcheck.log 2>&1; echo "initcheck rc=$?"; tail -4 $OUT/initcheck.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "bench N=1 rc=$?"; cut -c1-600 $OUT/bench_n1.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_n1.json 2> $OUT/bench_ref_n1.err; echo "bench ref rc=$?"; cut -c1-300 $OUT/bench_ref_n1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 4 --warmup 3 --skip-cpu --e2e-steps 0 > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fold_direct_kernel -s 20 -c 1 -o $OUT/fold_direct_full python bench.py --steps 4 --warmup 3 --skip-cpu --e2e-steps 0 > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"; ls -la $OUT/*.ncu-rep
