#!/bin/bash
# SM split for perfect covers at N=2 (pre-reduce HBM-bound)
bash tools/gpu_envab.sh 2 "RCV_PERFECT_SHARE=0" "RCV_PERFECT_SHARE=0.2" "RCV_PERFECT_SHARE=0.25" "RCV_PERFECT_SHARE=0.15" "RCV_PERFECT_SHARE=0"
