#!/bin/bash
# round-2 job H (1 GPU): 256-bit vector path -- parity, N=1 bench A/B, probe follow-up
OUT=gpurun_out/r2h; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fold.py tests/test_gpu_guards.py tests/test_gpu_commit.py tests/test_gpu_kacc.py -q -p no:randomly > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for W in 2 1 0; do
  RCV_W256=$W timeout 600 python bench.py --skip-cpu --e2e-steps 0 > $OUT/bench_n1_w$W.json 2> $OUT/bench_n1_w$W.err; echo "bench W256=$W rc=$?"
  python -c "
import json; d=json.loads(open('$OUT/bench_n1_w$W.json').read().strip().splitlines()[-1]); s=d['step_ms']; r=d['roofline']
print('  ms/step %.3f free %.3f fail %.3f deg %.3f parity %s launch %.1f us %.0f GB/s frac %.3f' % (d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity'], r['mean_launch_us'], r['achieved'], r['frac']))"
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/hbm_probe tools/hbm_probe.cu && PROBE_ONLY=1 timeout 600 /tmp/hbm_probe > $OUT/hbm_probe2.jsonl 2> $OUT/hbm_probe2.err; echo "probe rc=$?"; cat $OUT/hbm_probe2.jsonl
