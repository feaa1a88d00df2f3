#!/bin/bash
# round-2 job X (4 GPUs): configs[3] HSDP with the committed loss trajectory;
# merged timelines of the N=4 degraded layout and of N=2
OUT=gpurun_out/r2x; mkdir -p $OUT
timeout 900 python tools/hsdp_train.py --out $OUT/hsdp_configs3.json > $OUT/hsdp.log 2>&1; echo "hsdp rc=$?"; python -c "
import json; d=json.load(open('$OUT/hsdp_configs3.json')); print({k: d[k] for k in ('committed_loss_failure_free','committed_loss_with_failure','loss_trajectory_bitwise_equal','survivor_params_bitwise_equal_failure_free')})"
tr() { N=$1; tag=$2; shift 2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29700+RANDOM%200)) bench.py --gpus $N --steps 4 --warmup 5 --skip-cpu --e2e-steps 0 --trace /tmp/tr_$tag "$@" > /dev/null 2>&1
  files=""; for r in $(seq 0 $((N-1))); do files="$files /tmp/tr_${tag}_rank$r.json"; done
  (cd tools && python trace_merge.py $files) > $OUT/merge_$tag.txt 2>&1
  (cd tools && python trace_summary.py $files) > $OUT/summary_$tag.txt 2>&1; echo "trace $tag"; }
tr 4 n4deg --trace-degraded
tr 2 n2free
tr 2 n2deg --trace-degraded
