#!/bin/bash
# carveout default (-1) vs max-shared, and the perfect-cover share, with every
# other runtime default of the round's end
bash tools/gpu_envab.sh 4 "RCV_CARVEOUT=-1" "RCV_CARVEOUT=100" "RCV_CARVEOUT=-1 RCV_PERFECT_SHARE=0.35" "RCV_CARVEOUT=-1"
bash tools/gpu_envab.sh 2 "RCV_CARVEOUT=-1" "RCV_CARVEOUT=100" "RCV_CARVEOUT=-1 RCV_PERFECT_SHARE=0.35"
