#!/bin/bash
# round-2 job AB (4 GPUs): the new combine-share default at N=4 / N=2 (two
# reps each) with e2e, and the multi-GPU suite
OUT=gpurun_out/r2ab; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s e2e %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity'], (d.get('e2e') or {}).get('value')))"; }
P=30020
for rep in 1 2; do for N in 4 2; do P=$((P+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N > $OUT/bench_n${N}_rep$rep.json 2> $OUT/bench_n${N}_rep$rep.err; echo "bench N=$N rc=$?"; summ $OUT/bench_n${N}_rep$rep.json
done; done
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_hsdp.py tests/test_gpu_realkill.py -q -p no:randomly > $OUT/pytest_dist.log 2>&1; echo "pytest dist rc=$?"; tail -2 $OUT/pytest_dist.log
