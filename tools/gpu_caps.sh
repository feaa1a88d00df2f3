#!/bin/bash
# SM-partitioning sweep with the combine forced to DIRECT
for N in 4 2; do
bash tools/gpu_envab.sh $N "RCV_COMB_CTAS=0" "RCV_COMB_VARIANT=2" \
  "RCV_COMB_VARIANT=2 RCV_COMB_CTAS=0.35 RCV_PRE_CTAS=0.65" \
  "RCV_COMB_VARIANT=2 RCV_COMB_CTAS=0.25 RCV_PRE_CTAS=0.75" \
  "RCV_COMB_VARIANT=2 RCV_COMB_CTAS=0.5 RCV_PRE_CTAS=0.5" \
  "RCV_COMB_VARIANT=2 RCV_COMB_CTAS=0.35"
done
