#!/bin/bash
# N-GPU bench A/B over environment settings: bash gpu_envab.sh N "ENV=.." "ENV=.." ...
N=$1; shift; i=0
for E in "$@"; do
  i=$((i+1))
  env $E timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29800+i)) bench.py --gpus $N --steps 30 --warmup 5 --skip-cpu --e2e-steps 0 \
    2>/dev/null | grep "^{" > gpurun_out/envab_$i.json
  python3 -c "
import json; ls=[l for l in open('gpurun_out/envab_$i.json') if l.startswith('{')]
d=json.loads(ls[-1]); a=d['step_ms']['all']; k=d['kernels']
kd=d.get('kernels_degraded') or {}
f=lambda k: {n:(round(v['mean_launch_us']),round(v['nvlink_gbs_per_direction'] or 0)) for n,v in k.items()}
print('N$N [$E]', round(d['ms_per_step'],3), 'free', a[3], 'fail', round(d['step_ms']['failure_step'],2), 'post', a[-1], f(k), 'degraded', f(kd))" || echo "N$N [$E] failed"
done
