#!/bin/bash
# round-2 job AS (4 GPUs): e2e copy pipelining A/B at N=4 and N=1 on one box
OUT=gpurun_out/r2as; mkdir -p $OUT
e2e() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); e=d['e2e']; print('  e2e %.3f M tok/s  %.1f ms/step  %.1f GB/s per GPU' % (e['value']/1e6, e['ms_per_step'], e['pcie_gbs_per_gpu']))"; }
for MODE in pipelined serial pipelined serial; do
  BENCH_E2E_COPY=$MODE timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((30400+RANDOM%100)) bench.py --gpus 4 --skip-cpu --steps 4 --warmup 3 > $OUT/bench_n4_$MODE.json 2> $OUT/bench_n4_$MODE.err; echo "N=4 $MODE rc=$?"; e2e $OUT/bench_n4_$MODE.json
done
for MODE in pipelined serial; do
  CUDA_VISIBLE_DEVICES=0 BENCH_E2E_COPY=$MODE timeout 900 python bench.py --skip-cpu --steps 4 --warmup 3 > $OUT/bench_n1_$MODE.json 2> $OUT/bench_n1_$MODE.err; echo "N=1 $MODE rc=$?"; e2e $OUT/bench_n1_$MODE.json
done
nproc; lscpu | grep -i "model name\|socket\|numa node(s)"; nvidia-smi topo -m | head -8
