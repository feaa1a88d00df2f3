#!/bin/bash
# round-2 job AT (4 GPUs): copy-engine reduce-scatter (RCV_CE=1): parity suite, A/B at
# N=4 / N=2, repeated whole-rank deaths
OUT=gpurun_out/r2at; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))
print('  free', {k:(round(v['mean_launch_us'],1)) for k,v in d['kernels'].items()}, 'deg', {k:(round(v['mean_launch_us'],1)) for k,v in d['kernels_degraded'].items()})"; }
P=30210
run() { N=$1; shift; P=$((P+1)); tag=n${N}_$(echo "$@" | tr ' =' '_-')_$P; [ -z "$1" ] && tag=n${N}_default_$P
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --skip-cpu --e2e-steps 0 > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err; echo "bench N=$N $@ rc=$?"; summ $OUT/bench_$tag.json; tail -2 $OUT/bench_$tag.err | cut -c1-300; }
run 4 RCV_CE=1
run 4 RCV_CE=1 RCV_PRE_CTAS=0.75
run 4
run 2 RCV_CE=1
run 2
RCV_CE=1 timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_hsdp.py -q -p no:randomly -x > $OUT/pytest_dist_ce.log 2>&1; echo "pytest ce rc=$?"; tail -3 $OUT/pytest_dist_ce.log
RCV_CE=1 timeout 600 python tools/repeat_dist.py --world 4 --trials 50 --sizes 6464,2560064 --seed 91 --out $OUT/repeat_w4_ce.jsonl > $OUT/repeat_w4_ce.log 2>&1; echo "repeat ce rc=$?"; tail -1 $OUT/repeat_w4_ce.jsonl | cut -c1-150
