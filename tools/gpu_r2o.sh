#!/bin/bash
# round-2 job O (4 GPUs): merged multi-rank timeline of the N=4 pipeline and
# SM-share A/B of the overlapped kernels
OUT=gpurun_out/r2o; mkdir -p $OUT
trace() { tag=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29911+RANDOM%500)) bench.py --gpus 4 --steps 4 --warmup 5 --skip-cpu --e2e-steps 0 --trace /tmp/tr_$tag > /dev/null 2>&1
  (cd tools && python trace_merge.py /tmp/tr_${tag}_rank0.json /tmp/tr_${tag}_rank1.json /tmp/tr_${tag}_rank2.json /tmp/tr_${tag}_rank3.json) > $OUT/merge_$tag.txt 2>&1
  (cd tools && python trace_summary.py /tmp/tr_${tag}_rank0.json /tmp/tr_${tag}_rank3.json) > $OUT/summary_$tag.txt 2>&1
  echo "trace $tag done"
}
trace default
trace bcast25 RCV_BCAST_CTAS=0.25
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))"; }
P=29800
for CFG in "RCV_BCAST_CTAS=0.25" "RCV_BCAST_CTAS=0.15" "RCV_COMB_CTAS=0.4" "RCV_COMB_CTAS=0.4 RCV_PRE_CTAS=0.6" "RCV_BCAST_CTAS=0.25 RCV_COMB_CTAS=0.4"; do P=$((P+1))
  tag=$(echo $CFG | tr ' =' '_-')
  env $CFG timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --skip-cpu --e2e-steps 0 > $OUT/bench_n4_$tag.json 2> $OUT/bench_n4_$tag.err; echo "bench N=4 $CFG rc=$?"; summ $OUT/bench_n4_$tag.json
done
