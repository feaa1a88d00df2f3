#!/bin/bash
# N=4 timelines of the default runtime (failure-free and degraded layouts)
OUT=gpurun_out; mkdir -p $OUT
for D in "" "--trace-degraded"; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29913 bench.py --gpus 4 --steps 4 --warmup 5 --skip-cpu --e2e-steps 0 --trace $OUT/d4${D:+_deg} $D > /dev/null 2>&1
  echo "trace $D rc=$?"
done
