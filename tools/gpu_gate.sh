#!/bin/bash
# combine SM share of fragmented covers (post-failure layouts)
bash tools/gpu_envab.sh 4 "RCV_FRAG_SHARE=0.35" "RCV_FRAG_SHARE=0.5" "RCV_FRAG_SHARE=0.25"
bash tools/gpu_envab.sh 2 "RCV_FRAG_SHARE=0.35" "RCV_FRAG_SHARE=0.5" "RCV_FRAG_SHARE=0.25"
