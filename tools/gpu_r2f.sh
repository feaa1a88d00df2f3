#!/bin/bash
# round-2 job F (4 GPUs): NVLS multicast all-gather -- parity tests, then the
# N=4 / N=2 bench with and without RCV_MC=1.
OUT=gpurun_out/r2f; mkdir -p $OUT
python tools/nvls_probe.py > $OUT/nvls_probe.json 2>&1; echo "nvls rc=$?"
timeout 600 python -m pytest tests/test_gpu_dist.py -q -p no:randomly -k "True" > $OUT/pytest_mc.log 2>&1; echo "pytest mc rc=$?"; tail -5 $OUT/pytest_mc.log
for N in 4 2; do for MC in 0 1; do
  RCV_MC=$MC timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29620+N+MC)) bench.py --gpus $N --skip-cpu --e2e-steps 0 > $OUT/bench_n${N}_mc${MC}.json 2> $OUT/bench_n${N}_mc${MC}.err
  echo "bench N=$N MC=$MC rc=$?"; tail -2 $OUT/bench_n${N}_mc${MC}.err | cut -c1-300; python -c "
import json; d=json.loads(open('$OUT/bench_n${N}_mc${MC}.json').read().strip().splitlines()[-1]); s=d['step_ms']
print('ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))
print(' free', {k:(round(v['mean_launch_us'],1), round(v['nvlink_gbs_per_direction'] or 0)) for k,v in d['kernels'].items()})
print(' deg ', {k:(round(v['mean_launch_us'],1), round(v['nvlink_gbs_per_direction'] or 0)) for k,v in d['kernels_degraded'].items()})"
done; done
