#!/bin/bash
# Runtime schedule A/B on a 4-GPU box: per-plan broadcast stream vs side stream
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m multigpu -q -x > $OUT/pytest_multi_bs.log 2>&1; echo "pytest multigpu rc=$?"
tail -2 $OUT/pytest_multi_bs.log
bash tools/gpu_envab.sh 4 "RCV_BCAST_STREAM=1" "RCV_BCAST_STREAM=0" "RCV_BCAST_STREAM=1"
bash tools/gpu_envab.sh 2 "RCV_BCAST_STREAM=1" "RCV_BCAST_STREAM=0"
