#!/bin/bash
# round-2 job AQ (4 GPUs): push data flow with other SM shares at N=4
OUT=gpurun_out/r2aq; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))"; }
P=30200
run() { N=$1; shift; P=$((P+1)); tag=n${N}_$(echo "$@" | tr ' =' '_-')_$P; [ -z "$1" ] && tag=n${N}_default_$P
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --skip-cpu --e2e-steps 0 > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err; echo "bench N=$N $@ rc=$?"; summ $OUT/bench_$tag.json; }
run 4 RCV_PUSH=1 RCV_PRE_CTAS=0.75 RCV_COMB_CTAS=0.15
run 4 RCV_PUSH=1 RCV_PRE_CTAS=0.75 RCV_COMB_CTAS=0.1
run 4 RCV_PUSH=1 RCV_PRE_CTAS=0.9 RCV_COMB_CTAS=0.1
run 4 RCV_PUSH=1 RCV_PRE_CTAS=0.5 RCV_COMB_CTAS=0.1
