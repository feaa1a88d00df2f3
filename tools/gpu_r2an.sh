#!/bin/bash
# round-2 job AN (4 GPUs): merged timelines of the final N=4 schedule
OUT=gpurun_out/r2an; mkdir -p $OUT
tr() { N=$1; tag=$2; shift 2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29700+RANDOM%200)) bench.py --gpus $N --steps 4 --warmup 5 --skip-cpu --e2e-steps 0 --trace /tmp/tr_$tag "$@" > /dev/null 2>&1
  files=""; for r in $(seq 0 $((N-1))); do files="$files /tmp/tr_${tag}_rank$r.json"; done
  (cd tools && python trace_merge.py $files) > $OUT/merge_$tag.txt 2>&1
  (cd tools && python trace_summary.py $files) > $OUT/summary_$tag.txt 2>&1; echo "trace $tag"; }
tr 4 n4free
tr 4 n4deg --trace-degraded
