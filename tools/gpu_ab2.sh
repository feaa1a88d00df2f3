#!/bin/bash
# N-GPU A/B of the pre-reduce (--variant) and combine (--combine-variant) kernels
N=$1; shift; i=0
for V in "$@"; do
  set -- $V; i=$((i+1))
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29700+i)) bench.py --gpus $N --steps 30 --warmup 5 --skip-cpu --e2e-steps 0 \
    --variant $1 --combine-variant $2 2>/dev/null | grep "^{" > gpurun_out/ab_$i.json
  python3 -c "
import json; ls=[l for l in open('gpurun_out/ab_$i.json') if l.startswith('{')]
d=json.loads(ls[-1]); a=d['step_ms']['all']; k=d['kernels']
print('N$N v=$1 cv=$2', round(d['ms_per_step'],3), 'free', a[3], 'post', a[-1], {n:(round(v['mean_launch_us']),round(v['hbm_gbs']),round(v['nvlink_gbs_per_direction'] or 0)) for n,v in k.items()})" || echo "N$N $V failed"
done
