#!/bin/bash
# round-2 job R (4 GPUs): local-broadcast SM cap sweep at N=4 / N=2, merged
# timeline at the best N=4 setting
OUT=gpurun_out/r2r; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))"; }
P=29890
run() { N=$1; shift; P=$((P+1)); tag=n${N}_$(echo "$@" | tr ' =' '_-'); [ -z "$1" ] && tag=n${N}_default
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --skip-cpu --e2e-steps 0 > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err; echo "bench N=$N $@ rc=$?"; summ $OUT/bench_$tag.json; }
run 4 RCV_BCAST_CTAS=0.15
run 4 RCV_BCAST_CTAS=0.2
run 4 RCV_BCAST_CTAS=0.25
run 4 RCV_BCAST_CTAS=0.35
run 4 RCV_BCAST_CTAS=0.25 RCV_COMB_CTAS=0.3
run 4 RCV_BCAST_CTAS=0.25 RCV_PRE_CTAS=0.65
run 2 RCV_BCAST_CTAS=0.5
run 2 RCV_BCAST_CTAS=0.75
run 2
env RCV_BCAST_CTAS=0.25 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29990 bench.py --gpus 4 --steps 4 --warmup 5 --skip-cpu --e2e-steps 0 --trace /tmp/tr_r > /dev/null 2>&1
(cd tools && python trace_merge.py /tmp/tr_r_rank0.json /tmp/tr_r_rank1.json /tmp/tr_r_rank2.json /tmp/tr_r_rank3.json) > $OUT/merge_bcast25.txt 2>&1
(cd tools && python trace_summary.py /tmp/tr_r_rank0.json /tmp/tr_r_rank1.json /tmp/tr_r_rank2.json /tmp/tr_r_rank3.json) > $OUT/summary_bcast25.txt 2>&1
echo traced
