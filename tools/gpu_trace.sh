#!/bin/bash
# N-GPU timeline of 4 failure-free bench steps, summarised per rank
N=${1:-4}; shift
mkdir -p gpurun_out
env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29911 bench.py --gpus $N --steps 4 --warmup 5 --skip-cpu --e2e-steps 0 --trace /tmp/tr > /dev/null 2>&1
for r in 0 $((N-1)); do python tools/trace_summary.py /tmp/tr_rank$r.json; done
python tools/trace_summary.py --timeline /tmp/tr_rank0.json
