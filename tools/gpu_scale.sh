#!/bin/bash
# 4-GPU box job: multi-GPU parity tests, bench at N=2 and N=4 (plus the
# reference arm), then N=4 timelines (failure-free and degraded layouts).
# usage: bash tools/gpu_scale.sh TAG
TAG=${1:-scale}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu4_$TAG.log 2>&1; echo "pytest gpu rc=$?"
tail -3 $OUT/pytest_gpu4_$TAG.log
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port $((29600+N)) bench.py --gpus $N > $OUT/bench_n${N}_$TAG.json 2> $OUT/bench_n${N}_$TAG.err
  echo "bench N=$N rc=$?"; cut -c1-400 $OUT/bench_n${N}_$TAG.json
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port $((29700+N)) bench.py --gpus $N --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_n${N}_$TAG.json 2> $OUT/bench_ref_n${N}_$TAG.err
  echo "ref N=$N rc=$?"; cut -c1-300 $OUT/bench_ref_n${N}_$TAG.json
done
if [ "$TRACE" = "1" ]; then
for D in "" "--trace-degraded"; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29913 bench.py --gpus 4 --steps 4 --warmup 5 --skip-cpu --e2e-steps 0 --trace $OUT/t4${D:+_deg} $D > /dev/null 2>&1
  echo "trace $D rc=$?"
done
fi
