#!/bin/bash
# gated runtime (with the per-plan broadcast stream) vs barrier runtime
OUT=gpurun_out; mkdir -p $OUT
RCV_GATE=1 timeout 600 python -m pytest tests -m multigpu -q -x > $OUT/pytest_multi_g.log 2>&1; echo "pytest multigpu (gate) rc=$?"
tail -2 $OUT/pytest_multi_g.log
bash tools/gpu_envab.sh 4 "RCV_GATE=1" "RCV_GATE=0" "RCV_GATE=1" "RCV_GATE=0"
bash tools/gpu_envab.sh 2 "RCV_GATE=1" "RCV_GATE=0"
