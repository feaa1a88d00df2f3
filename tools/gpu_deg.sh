#!/bin/bash
timeout 300 python bench.py --steps 6 --warmup 3 --skip-cpu --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N1', d['ms_per_step'], d['kernels'], d['kernels_degraded'])"
bash tools/gpu_envab.sh 2 "RCV_X=0"
bash tools/gpu_envab.sh 4 "RCV_X=0"
