#!/bin/bash
# N=2 timelines: failure-free and degraded layouts
for D in "" "--trace-degraded"; do
echo "=== N=2 $D"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29913 bench.py --gpus 2 --steps 4 --warmup 5 --skip-cpu --e2e-steps 0 --trace /tmp/t2 $D > /dev/null 2>&1
python tools/trace_summary.py /tmp/t2_rank0.json /tmp/t2_rank1.json | grep -E "mean|busy|gaps"
python tools/trace_summary.py --timeline /tmp/t2_rank0.json | head -24
done
