#!/bin/bash
# Sweep the native runtime's CTA caps on N GPUs (one bench line per setting).
# usage: bash gpu_sweep.sh N "PRE COMB BCAST" ...
N=$1; shift
OUT=gpurun_out; mkdir -p $OUT
i=0
for cfg in "$@"; do
  set -- $cfg
  i=$((i+1))
  RCV_PRE_CTAS=$1 RCV_COMB_CTAS=$2 RCV_BCAST_CTAS=$3 timeout 300 python -m torch.distributed.run \
    --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600+i)) bench.py \
    --gpus $N --steps 30 --warmup 5 --skip-cpu --e2e-steps 0 > $OUT/sweep_$i.json 2>/dev/null
  python3 -c "
import json,sys
d=json.loads([l for l in open('$OUT/sweep_$i.json') if l.startswith('{')][-1])
k=d['kernels']
print('cfg=[$cfg] ms/step %.3f' % d['ms_per_step'], ' '.join('%s:%.0fus' % (n, v['mean_launch_us']) for n, v in k.items()), 'comb nvl/dir %.0f' % k['combine']['nvlink_gbs_per_direction'])
" || echo "cfg=[$cfg] failed"
done
