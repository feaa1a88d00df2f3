#!/bin/bash
# barrier / SM-partitioning experiments at N=4: step A/B then traces
bash tools/gpu_envab.sh 4 "RCV_BAR_FENCE=1" "RCV_BAR_FENCE=0" "RCV_COMB_CTAS=0.5" "RCV_COMB_CTAS=0.35 RCV_PRE_CTAS=0.65" "RCV_PRE_CTAS=0.5"
for E in "RCV_BAR_FENCE=0" "RCV_COMB_CTAS=0.5"; do
  echo "== trace $E"
  bash tools/gpu_trace.sh 4 $E 2>&1 | grep -E "mean|busy|gaps" | head -12
done
