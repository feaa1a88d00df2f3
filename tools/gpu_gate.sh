#!/bin/bash
# two vectors per thread in the DIRECT perfect-tree combine
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m multigpu -q -x > $OUT/pytest_multi_pair.log 2>&1; echo "pytest multigpu rc=$?"
tail -2 $OUT/pytest_multi_pair.log
bash tools/gpu_envab.sh 4 "RCV_PAIR=1" "RCV_PAIR=0" "RCV_PAIR=1" "RCV_PAIR=0"
bash tools/gpu_envab.sh 2 "RCV_PAIR=1" "RCV_PAIR=0"
