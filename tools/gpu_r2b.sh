#!/bin/bash
# round-2 job B (2 GPUs): GPU tests, repeats, N=1/N=2 bench, real-kill
# recovery, GPT-2 K-ACC training, NVLS probe.
OUT=gpurun_out/r2b; mkdir -p $OUT
nvidia-smi -L > $OUT/gpus.txt
python tools/nvls_probe.py > $OUT/nvls_probe.json 2>&1; echo "nvls rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 $OUT/pytest_gpu.log | grep -v "^$"
timeout 120 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "bench N=1 rc=$?"; cut -c1-600 $OUT/bench_n1.json; tail -3 $OUT/bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "bench N=2 rc=$?"; cut -c1-600 $OUT/bench_n2.json; tail -3 $OUT/bench_n2.err
timeout 600 python tools/realkill_bench.py --world 2 --out $OUT/realkill_w2.json > $OUT/realkill_w2.log 2>&1; echo "realkill rc=$?"; tail -c 1500 $OUT/realkill_w2.log
for W in 4 8; do for R in 1 0; do
  S=6464,2560064; [ $W = 8 ] && S=6464
  RCV_REUSE=$R timeout 900 python tools/repeat_dist.py --world $W --trials 100 --sizes $S --seed $((W*10+R)) --out $OUT/repeat_w${W}_reuse${R}.jsonl > $OUT/repeat_w${W}_reuse${R}.log 2>&1
  echo "repeat W=$W REUSE=$R rc=$?"; tail -1 $OUT/repeat_w${W}_reuse${R}.log
done; done
timeout 900 python tools/gpt2_train.py --out $OUT/gpt2_kacc.json > $OUT/gpt2.log 2>&1; echo "gpt2 rc=$?"; tail -c 1200 $OUT/gpt2.log
