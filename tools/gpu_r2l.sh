#!/bin/bash
# round-2 job L (4 GPUs): barrier lag (barriers on their own stream, overlapping
# the previous combine) A/B at N=4 / N=2, multi-GPU suite
OUT=gpurun_out/r2l; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s host %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity'], d.get('host_step_ms')))
print('  prof', d.get('host_prof_ms_per_step'))
print('  free', {k:(round(v['mean_launch_us'],1), round(v['hbm_gbs'] or 0), round(v['nvlink_gbs_per_direction'] or 0)) for k,v in d['kernels'].items()})
print('  deg ', {k:(round(v['mean_launch_us'],1), round(v['hbm_gbs'] or 0), round(v['nvlink_gbs_per_direction'] or 0)) for k,v in d['kernels_degraded'].items()})"; }
for N in 4 2; do for LAG in 2 1; do
  RCV_BARRIER_LAG=$LAG timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29650+N+LAG*10)) bench.py --gpus $N --skip-cpu --e2e-steps 0 > $OUT/bench_n${N}_lag$LAG.json 2> $OUT/bench_n${N}_lag$LAG.err; echo "bench N=$N lag=$LAG rc=$?"; summ $OUT/bench_n${N}_lag$LAG.json
done; done
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_hsdp.py tests/test_gpu_realkill.py -q -p no:randomly > $OUT/pytest_dist.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_dist.log
