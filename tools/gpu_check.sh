#!/bin/bash
# GPU-box job: parity tests, smoke, bench, then (only if the bench exited 0)
# the ncu launch list and one full capture of the dominant kernel.
# usage: bash tools/gpu_check.sh TAG [bench args...]
TAG=${1:-r1}; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest_gpu_$TAG.log
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 120 python __graft_entry__.py smoke > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/smoke_$TAG.log
BENCH="python bench.py $*"
timeout 600 $BENCH > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; RC=$?
echo "bench rc=$RC"; cat $OUT/bench_$TAG.json; tail -3 $OUT/bench_$TAG.err
if [ "$NCU" = "1" ] && [ $RC = 0 ]; then
  SMALL="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --skip-cpu $NCU_ARGS"
  timeout 300 $SMALL > $OUT/ncu_plain_$TAG.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_$TAG.csv $SMALL > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-fold_} \
      -s ${NCU_S:-40} -c 1 -o $OUT/prof_$TAG $SMALL > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
  tail -2 $OUT/ncu_full_$TAG.log
fi
