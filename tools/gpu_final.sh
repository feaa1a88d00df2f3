#!/bin/bash
# end-of-round 4-GPU job: copy-engine all-gather check, then parity + benches
bash tools/gpu_envab.sh 4 "RCV_CE_GATHER=1" "RCV_CE_GATHER=0"
bash tools/gpu_scale.sh s5
