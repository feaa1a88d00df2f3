#!/bin/bash
bash tools/gpu_multi.sh caps4 4
bash tools/gpu_envab.sh 2 "RCV_COMB_CTAS=0.35"
bash tools/gpu_trace.sh 4 2>&1 | grep -E "mean|busy|gaps" | head -12
