#!/bin/bash
bash tools/gpu_multi.sh w4 4
bash tools/gpu_envab.sh 2 "RCV_X=0" "RCV_X=1"
bash tools/gpu_envab.sh 4 "RCV_X=0"
