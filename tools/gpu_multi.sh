#!/bin/bash
# GPU-box job on N GPUs: multi-GPU tests, then the N-rank bench via torchrun.
# usage: bash gpu_multi.sh TAG N [bench args...]
TAG=$1; N=$2; shift 2
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi topo -m > $OUT/topo_$TAG.txt 2>&1
timeout 600 python -m pytest tests -m multigpu -q -x > $OUT/pytest_multi_$TAG.log 2>&1; echo "pytest multigpu rc=$?"
tail -3 $OUT/pytest_multi_$TAG.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
   --master-port 29511 bench.py --gpus $N "$@" > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
echo "bench rc=$?"; cat $OUT/bench_$TAG.json; grep -v Warning $OUT/bench_$TAG.err | tail -5
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
   --master-port 29512 bench.py --gpus $N --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_$TAG.json 2>&1
echo "ref rc=$?"; tail -2 $OUT/bench_ref_$TAG.json
