#!/bin/bash
# round-2 job AV (4 GPUs): multicast for the node-heaviest rank of fragmented
# covers only (RCV_MC=2) vs unicast: A/B at N=4 / N=2 and the parity suite
OUT=gpurun_out/r2av; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))
print('  deg', {k:(round(v['mean_launch_us'],1)) for k,v in d['kernels_degraded'].items()})"; }
P=30230
run() { N=$1; shift; P=$((P+1)); tag=n${N}_$(echo "$@" | tr ' =' '_-')_$P; [ -z "$1" ] && tag=n${N}_default_$P
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --skip-cpu --e2e-steps 0 > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err; echo "bench N=$N $@ rc=$?"; summ $OUT/bench_$tag.json; tail -1 $OUT/bench_$tag.err | cut -c1-200; }
run 4 RCV_MC=2
run 4
run 4 RCV_MC=2
run 4
run 2 RCV_MC=2
run 2
RCV_MC=2 timeout 1200 python -m pytest tests/test_gpu_dist.py -q -p no:randomly -x > $OUT/pytest_dist_mc2.log 2>&1; echo "pytest mc2 rc=$?"; tail -2 $OUT/pytest_dist_mc2.log
