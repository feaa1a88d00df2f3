#!/bin/bash
# round-2 job D (4 GPUs): the GPU suite with one GPU per rank, N=4/N=2 bench,
# configs[3] HSDP (FSDP2 2 shards x 2 replicas), real-kill at 4 ranks,
# per-rank repeats, and NVLink counters of the N=4 combine covers.
OUT=gpurun_out/r2d; mkdir -p $OUT
nvidia-smi -L > $OUT/gpus.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:randomly > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -12 $OUT/pytest_gpu.log | grep -v "^$"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 4 > $OUT/bench_n4.json 2> $OUT/bench_n4.err; echo "bench N=4 rc=$?"; cut -c1-400 $OUT/bench_n4.json; tail -3 $OUT/bench_n4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 2 > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "bench N=2 rc=$?"; cut -c1-400 $OUT/bench_n2.json
timeout 900 python tools/hsdp_train.py --out $OUT/hsdp_configs3.json > $OUT/hsdp.log 2>&1; echo "hsdp rc=$?"; tail -c 1500 $OUT/hsdp.log
timeout 600 python tools/realkill_bench.py --world 4 --out $OUT/realkill_w4.json > $OUT/realkill_w4.log 2>&1; echo "realkill4 rc=$?"; tail -c 1200 $OUT/realkill_w4.log
for R in 1 0; do
  RCV_REUSE=$R timeout 600 python tools/repeat_dist.py --world 4 --trials 50 --sizes 6464,2560064 --seed $((40+R)) --out $OUT/repeat_w4_reuse${R}.jsonl > $OUT/repeat_w4_reuse${R}.log 2>&1
  echo "repeat W=4 REUSE=$R rc=$?"; tail -c 300 $OUT/repeat_w4_reuse${R}.log
done
for C in perfect 9 12 15; do timeout 120 python tools/ncu_combine.py --cover $C >> $OUT/combine_4gpu.jsonl 2>> $OUT/combine_4gpu.err; done; cat $OUT/combine_4gpu.jsonl
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:fold_ --csv python tools/ncu_combine.py --cover perfect --reps 1 > $OUT/ncu_combine_perfect.csv 2> $OUT/ncu_combine_perfect.err; echo "ncu perfect rc=$?"
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:fold_ --csv python tools/ncu_combine.py --cover 15 --reps 1 > $OUT/ncu_combine_15.csv 2> $OUT/ncu_combine_15.err; echo "ncu 15 rc=$?"
