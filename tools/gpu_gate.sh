#!/bin/bash
# combine variant / CTA count A/B on a 4-GPU box (perfect covers: DIRECT by AUTO)
bash tools/gpu_envab.sh 4 "RCV_COMB_VARIANT=0" "RCV_COMB_VARIANT=1"
bash tools/gpu_envab.sh 2 "RCV_COMB_VARIANT=0" "RCV_COMB_VARIANT=1"
