#!/bin/bash
# round-2 job AG (4 GPUs): the one-copy broadcast fused into the pre-reduce
# forest (RCV_BCAST_FUSE=1): parity suite and A/B at N=4
OUT=gpurun_out/r2ag; mkdir -p $OUT
RCV_BCAST_FUSE=1 timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_hsdp.py -q -p no:randomly > $OUT/pytest_dist_fuse.log 2>&1; echo "pytest fuse rc=$?"; tail -2 $OUT/pytest_dist_fuse.log
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))"; }
P=30100
run() { N=$1; shift; P=$((P+1)); tag=n${N}_$(echo "$@" | tr ' =' '_-')_$P; [ -z "$1" ] && tag=n${N}_default_$P
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --skip-cpu --e2e-steps 0 > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err; echo "bench N=$N $@ rc=$?"; summ $OUT/bench_$tag.json; }
for rep in 1 2; do
run 4
run 4 RCV_BCAST_FUSE=1
done
run 4 RCV_BCAST_FUSE=1 RCV_PRE_CTAS=0.7
run 4 RCV_BCAST_FUSE=1 RCV_PRE_CTAS=0.5
RCV_BCAST_FUSE=1 RCV_REUSE=0 timeout 600 python tools/repeat_dist.py --world 4 --trials 50 --sizes 6464,2560064 --seed 77 --out $OUT/repeat_w4_fuse.jsonl > $OUT/repeat_w4_fuse.log 2>&1; echo "repeat fuse rc=$?"; tail -1 $OUT/repeat_w4_fuse.jsonl | cut -c1-200
