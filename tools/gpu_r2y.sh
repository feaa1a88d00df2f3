#!/bin/bash
# round-2 job Y (4 GPUs): pool-set count (pre-reduce run-ahead) at N=4 / N=2
OUT=gpurun_out/r2y; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))"; }
P=29960
run() { N=$1; shift; P=$((P+1)); tag=n${N}_$(echo "$@" | tr ' =' '_-')_$P; [ -z "$1" ] && tag=n${N}_default_$P
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --skip-cpu --e2e-steps 0 > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err; echo "bench N=$N $@ rc=$?"; summ $OUT/bench_$tag.json; }
for rep in 1 2; do
run 4
run 4 RCV_POOL_SETS=6
run 4 RCV_POOL_SETS=8
done
run 2
run 2 RCV_POOL_SETS=6
