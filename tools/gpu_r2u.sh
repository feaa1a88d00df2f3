#!/bin/bash
# round-2 job U (4 GPUs): bucket-count sensitivity at N=4 (per-bucket
# overhead), full GPU suite with every device visible
OUT=gpurun_out/r2u; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))
print('  free', {k:(round(v['mean_launch_us'],1), round(v['hbm_gbs'] or 0), round(v['nvlink_gbs_per_direction'] or 0)) for k,v in d['kernels'].items()})"; }
P=29930
for K in 10 5 40; do P=$((P+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --skip-cpu --e2e-steps 0 --buckets $K > $OUT/bench_n4_K$K.json 2> $OUT/bench_n4_K$K.err; echo "bench N=4 K=$K rc=$?"; summ $OUT/bench_n4_K$K.json
done
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > $OUT/pytest_gpu_4gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu_4gpu.txt
