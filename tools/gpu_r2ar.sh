#!/bin/bash
# round-2 job AR (4 GPUs): the driver's scaling sequence on the final build,
# default arguments: N=1, 2, 4 (ours, then the reference arm), as
# `python -m torch.distributed.run ... bench.py --gpus N`
OUT=gpurun_out/r2ar; mkdir -p $OUT
for N in 1 2 4; do
  if [ $N = 1 ]; then
    CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "ours N=1 rc=$?"
    CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference > $OUT/ref_n1.json 2> $OUT/ref_n1.err; echo "ref N=1 rc=$?"
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((30300+N)) bench.py --gpus $N > $OUT/bench_n$N.json 2> $OUT/bench_n$N.err; echo "ours N=$N rc=$?"
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((30310+N)) bench.py --gpus $N --impl reference > $OUT/ref_n$N.json 2> $OUT/ref_n$N.err; echo "ref N=$N rc=$?"
  fi
  python -c "
import json
d=json.loads(open('$OUT/bench_n$N.json').read().strip().splitlines()[-1]); r=json.loads(open('$OUT/ref_n$N.json').read().strip().splitlines()[-1])
print('  N=$N ours %.2f M tok/s %.3f ms/step parity %s roof %.3f e2e %.3f M | ref %.3f M (cores %s)' % (d['value']/1e6, d['ms_per_step'], d['parity'], d['roofline']['frac'], d['e2e']['value']/1e6, r['value']/1e6, r['cpu_baseline']['cores']))"
done
