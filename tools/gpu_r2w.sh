#!/bin/bash
# round-2 job W (4 GPUs): re-verify the reworked synchronisation (barrier
# stream, lag 2, four pool sets, stamps in the barrier kernel): repeated
# whole-rank deaths at W=4 and W=2, real-kill recovery at 4 ranks, configs[3]
# HSDP training, the full-size configs[1] commit test
OUT=gpurun_out/r2w; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_commit.py -q -p no:randomly -k full_size > $OUT/pytest_full_size.log 2>&1; echo "full-size rc=$?"; tail -2 $OUT/pytest_full_size.log
for W in 4 2; do for R in 1 0; do
  RCV_REUSE=$R timeout 900 python tools/repeat_dist.py --world $W --trials 100 --sizes 6464,2560064 --seed $((60+W+R)) --out $OUT/repeat_w${W}_reuse${R}.jsonl > $OUT/repeat_w${W}_reuse${R}.log 2>&1
  echo "repeat W=$W REUSE=$R rc=$?"; tail -1 $OUT/repeat_w${W}_reuse${R}.jsonl | cut -c1-300
done; done
timeout 600 python tools/realkill_bench.py --world 4 --out $OUT/realkill_w4.json > $OUT/realkill_w4.log 2>&1; echo "realkill4 rc=$?"; tail -c 1000 $OUT/realkill_w4.log
timeout 900 python tools/hsdp_train.py --out $OUT/hsdp_configs3.json > $OUT/hsdp.log 2>&1; echo "hsdp rc=$?"; tail -c 800 $OUT/hsdp.log
