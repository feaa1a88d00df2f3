#!/bin/bash
# committed-bucket reuse after a boundary: parity (all GPU tests) + A/B
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_reuse.log 2>&1; echo "pytest gpu rc=$?"
tail -2 $OUT/pytest_gpu_reuse.log
for R in 1 0; do
  RCV_REUSE=$R timeout 300 python bench.py --steps 30 --warmup 5 --skip-cpu --e2e-steps 0 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['step_ms']
print('N1 [RCV_REUSE=$R]', round(d['ms_per_step'],3), 'free', round(s['failure_free_median'],3), 'fail', round(s['failure_step'],3), 'post', round(s['degraded_median'],3), 'recovery', round(d['recovery_ms'],3))"
done
bash tools/gpu_envab.sh 4 "RCV_REUSE=1" "RCV_REUSE=0"
bash tools/gpu_envab.sh 2 "RCV_REUSE=1" "RCV_REUSE=0"
