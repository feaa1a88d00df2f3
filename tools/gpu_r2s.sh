#!/bin/bash
# round-2 job S (4 GPUs): barrier fence modes at N=4 / N=2 (new broadcast cap
# default), repeated for noise
OUT=gpurun_out/r2s; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))"; }
P=29910
run() { N=$1; shift; P=$((P+1)); tag=n${N}_$(echo "$@" | tr ' =' '_-')_$P; [ -z "$1" ] && tag=n${N}_default_$P
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --skip-cpu --e2e-steps 0 > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err; echo "bench N=$N $@ rc=$?"; summ $OUT/bench_$tag.json; }
for rep in 1 2; do
run 4
run 4 RCV_BARRIER_LEAN=1
run 4 RCV_BARRIER_LEAN=2
done
run 2
run 2 RCV_BARRIER_LEAN=1
run 2 RCV_BARRIER_LEAN=2
env RCV_BARRIER_LEAN=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29990 bench.py --gpus 4 --steps 4 --warmup 5 --skip-cpu --e2e-steps 0 --trace /tmp/tr_s > /dev/null 2>&1
(cd tools && python trace_merge.py /tmp/tr_s_rank0.json /tmp/tr_s_rank1.json /tmp/tr_s_rank2.json /tmp/tr_s_rank3.json) > $OUT/merge_lean1.txt 2>&1
echo traced
