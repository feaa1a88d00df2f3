#!/bin/bash
# round-2 job M (4 GPUs): barrier lag x pool sets A/B at N=4 / N=2
OUT=gpurun_out/r2m; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))
print('  prof', d.get('host_prof_ms_per_step'))"; }
P=29700
for N in 4 2; do for CFG in "1 3" "1 4" "2 4" "2 3"; do set -- $CFG; P=$((P+1))
  RCV_BARRIER_LAG=$1 RCV_POOL_SETS=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --skip-cpu --e2e-steps 0 > $OUT/bench_n${N}_L$1_S$2.json 2> $OUT/bench_n${N}_L$1_S$2.err; echo "bench N=$N lag=$1 sets=$2 rc=$?"; summ $OUT/bench_n${N}_L$1_S$2.json
done; done
