#!/bin/bash
# combine vector width A/B on a 4-GPU box
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m multigpu -q -x > $OUT/pytest_multi_w.log 2>&1; echo "pytest multigpu rc=$?"
tail -2 $OUT/pytest_multi_w.log
bash tools/gpu_envab.sh 2 "RCV_WIDE_COMB=1" "RCV_WIDE_COMB=0" "RCV_WIDE_COMB=2"
bash tools/gpu_envab.sh 4 "RCV_WIDE_COMB=1" "RCV_WIDE_COMB=0" "RCV_WIDE_COMB=2"
