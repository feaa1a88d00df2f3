#!/bin/bash
# round-2 job AM (4 GPUs): TMA-ring combine (cp.async.bulk loads of the peers'
# partials) vs the DIRECT pair kernel, N=4 / N=2
OUT=gpurun_out/r2am; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))
print('  free', {k:(round(v['mean_launch_us'],1), round(v['nvlink_gbs_per_direction'] or 0)) for k,v in d['kernels'].items()}, 'deg', {k:(round(v['mean_launch_us'],1)) for k,v in d['kernels_degraded'].items()})"; }
P=30160
run() { N=$1; shift; P=$((P+1)); tag=n${N}_$(echo "$@" | tr ' =-' '___')_$P
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --skip-cpu --e2e-steps 0 "$@" > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err; echo "bench N=$N $@ rc=$?"; summ $OUT/bench_$tag.json; }
run 4
run 4 --combine-variant 1
run 2
run 2 --combine-variant 1
