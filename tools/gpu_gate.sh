#!/bin/bash
# link-balanced owner slices at N=2 (degraded cover 4 + 2 nodes)
bash tools/gpu_envab.sh 2 "RCV_SLICE_BALANCE=1" "RCV_SLICE_BALANCE=0" "RCV_SLICE_BALANCE=1 RCV_SLICE_SHARE=0" "RCV_SLICE_BALANCE=0"
