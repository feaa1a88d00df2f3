#!/bin/bash
# round-2 job I (4 GPUs): GPU suite after the 256-bit path, N=4 / N=2 bench
# (256-bit pre-reduce forests and broadcasts), combine A/B, configs[2] sweep.
OUT=gpurun_out/r2i; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -p no:randomly > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_gpu.log
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s host %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity'], d.get('host_step_ms')))
print('  free', {k:(round(v['mean_launch_us'],1), round(v['hbm_gbs'] or 0), round(v['nvlink_gbs_per_direction'] or 0)) for k,v in d['kernels'].items()})
print('  deg ', {k:(round(v['mean_launch_us'],1), round(v['hbm_gbs'] or 0), round(v['nvlink_gbs_per_direction'] or 0)) for k,v in d['kernels_degraded'].items()})
print('  e2e', d.get('e2e'))"; }
for N in 4 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29630+N)) bench.py --gpus $N > $OUT/bench_n$N.json 2> $OUT/bench_n$N.err; echo "bench N=$N rc=$?"; summ $OUT/bench_n$N.json
done
for V in "RCV_W256=0" "RCV_W256_COMB=1"; do
  env $V timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29640 bench.py --gpus 4 --skip-cpu --e2e-steps 0 > $OUT/bench_n4_$V.json 2> $OUT/bench_n4_$V.err; echo "bench N=4 [$V] rc=$?"; summ $OUT/bench_n4_$V.json
done
timeout 900 python tools/sweep.py --n 2,4 --out $OUT/sweep_4gpu.jsonl > $OUT/sweep.log 2>&1; echo "sweep rc=$?"; tail -3 $OUT/sweep.log
