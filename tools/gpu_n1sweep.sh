#!/bin/bash
# N=1 kernel-variant sweep: one bench line per (env, args) setting
OUT=gpurun_out; mkdir -p $OUT; i=0
while [ $# -gt 0 ]; do
  i=$((i+1)); ENVS=$1; ARGS=$2; shift 2
  env $ENVS timeout 300 python bench.py --steps 20 --warmup 3 --skip-cpu --e2e-steps 0 $ARGS > $OUT/n1_$i.json 2>/dev/null
  python3 -c "
import json
d=json.loads([l for l in open('$OUT/n1_$i.json') if l.startswith('{')][-1])
r=d['roofline']; print('[$ENVS] [$ARGS] ms/step %.3f fused %.1f us  %.0f GB/s frac %.3f' % (d['ms_per_step'], r['mean_launch_us'], r['achieved'], r['frac']))" || echo "[$ENVS] [$ARGS] failed"
done
