#!/bin/bash
# round-2 job A (2 GPUs): GPU tests (multi-process ones share or span the
# GPUs), then the whole-rank-death repeats at 8 and 4 ranks, REUSE on/off.
OUT=gpurun_out/r2a; mkdir -p $OUT
nvidia-smi -L > $OUT/gpus.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:randomly > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest_gpu.log
tail -5 $OUT/pytest_gpu.log
timeout 120 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/smoke.log
for W in 8 4; do for R in 1 0; do
  RCV_REUSE=$R timeout 1200 python tools/repeat_dist.py --world $W --trials ${TRIALS:-100} --seed $((W*10+R)) --out $OUT/repeat_w${W}_reuse${R}.jsonl > $OUT/repeat_w${W}_reuse${R}.log 2>&1
  echo "repeat W=$W REUSE=$R rc=$?"; tail -1 $OUT/repeat_w${W}_reuse${R}.log
done; done
