#!/bin/bash
# fused per-bucket kernel: parity on the multi-GPU tests, then bench A/B
N=${1:-4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/fused_test.log 2>&1
grep -E "Error|assert|passed|failed" gpurun_out/fused_test.log | grep -v "TCPStore\|sendBytes\|should dump\|frame #" | head -20
bash tools/gpu_envab.sh $N "RCV_FUSED=0" "RCV_FUSED=1" "RCV_FUSED=1 RCV_FUSED_A=0.6"
bash tools/gpu_envab.sh 2 "RCV_FUSED=0" "RCV_FUSED=1"
