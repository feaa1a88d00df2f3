#!/bin/bash
# round-2 job AL (4 GPUs): ncu --set full of the N=4 perfect-cover combine
# (fold_direct_pair_kernel<ProgFull<2>>, one process over 4 GPUs, the same
# kernel and access pattern as the multi-process combine) plus NVLink
# counters of the degraded cover 15
OUT=gpurun_out/r2al; mkdir -p $OUT
timeout 300 python tools/ncu_combine.py --cover perfect > $OUT/combine_perfect.json 2>&1; echo "combine rc=$?"; cat $OUT/combine_perfect.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fold_direct_pair -c 1 -o $OUT/combine_pair_full python tools/ncu_combine.py --cover perfect --reps 1 > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"; ls -la $OUT/*.ncu-rep
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:fold_ --csv python tools/ncu_combine.py --cover 15 --reps 1 > $OUT/ncu_combine_15.csv 2> $OUT/ncu_combine_15.err; echo "ncu 15 rc=$?"
