#!/bin/bash
# round-2 job C (2 GPUs)
OUT=gpurun_out/r2c; mkdir -p $OUT
python tools/nvls_probe.py > $OUT/nvls_probe.json 2>&1; echo "nvls rc=$?"; python -c "import json;d=json.load(open('$OUT/nvls_probe.json'));print(d.get('granularity'), d.get('multicast_object'))"
timeout 900 python -m pytest tests -m gpu -q -p no:randomly > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 $OUT/pytest_gpu.log | grep -v "^$"
timeout 600 python tools/realkill_bench.py --world 2 --out $OUT/realkill_w2.json > $OUT/realkill_w2.log 2>&1; echo "realkill rc=$?"; tail -c 1800 $OUT/realkill_w2.log
for W in 4 8; do for R in 1 0; do
  S=6464,2560064; [ $W = 8 ] && S=6464
  RCV_REUSE=$R timeout 900 python tools/repeat_dist.py --world $W --trials 100 --sizes $S --seed $((W*10+R)) --out $OUT/repeat_w${W}_reuse${R}.jsonl > $OUT/repeat_w${W}_reuse${R}.log 2>&1
  echo "repeat W=$W REUSE=$R rc=$?"; tail -c 400 $OUT/repeat_w${W}_reuse${R}.log
done; done
timeout 600 python bench.py --skip-cpu --e2e-steps 0 > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "bench N=1 rc=$?"; cut -c1-300 $OUT/bench_n1.json
for V in "" "RCV_NO_STAMPS=1" "RCV_STAMP_KERNEL=1" "RCV_NO_FIXED=1"; do
  env $V timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --skip-cpu --e2e-steps 0 > $OUT/bench_n2_${V:-default}.json 2> $OUT/bench_n2_${V:-default}.err
  echo "bench N=2 [$V] rc=$?"; python -c "
import json,sys; d=json.loads(open('$OUT/bench_n2_${V:-default}.json').read().strip().splitlines()[-1]); s=d['step_ms']
print('ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))
print(' free', {k:(round(v['mean_launch_us'],1), round(v['nvlink_gbs_per_direction'] or 0)) for k,v in d['kernels'].items()})
print(' deg ', {k:(round(v['mean_launch_us'],1), round(v['nvlink_gbs_per_direction'] or 0)) for k,v in d['kernels_degraded'].items()})"
done
for C in perfect 2 3 4 5; do timeout 120 python tools/ncu_combine.py --cover $C >> $OUT/combine_2gpu.jsonl 2>> $OUT/combine_2gpu.err; done; cat $OUT/combine_2gpu.jsonl
