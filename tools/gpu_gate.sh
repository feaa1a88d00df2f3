#!/bin/bash
# PDL combine (launched as a programmatic dependent of its barrier) A/B
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m multigpu -q -x > $OUT/pytest_multi_pdl.log 2>&1; echo "pytest multigpu rc=$?"
tail -2 $OUT/pytest_multi_pdl.log
bash tools/gpu_envab.sh 4 "RCV_PDL=1" "RCV_PDL=0" "RCV_PDL=1" "RCV_PDL=0"
bash tools/gpu_envab.sh 2 "RCV_PDL=1" "RCV_PDL=0"
