#!/bin/bash
# round-2 job Q (4 GPUs): stamps written by the barrier kernel (no stream
# memops): N=4/N=2 bench vs no-stamps, SM-share A/B, multi-GPU suite
OUT=gpurun_out/r2q; mkdir -p $OUT
summ() { python -c "
import json; d=json.loads(open('$1').read().strip().splitlines()[-1]); s=d['step_ms']
print('  %.2f M ms/step %.3f free %.3f fail %.3f deg %.3f parity %s' % (d['value']/1e6, d['ms_per_step'], s['failure_free_median'], s['failure_step'], s['degraded_median'], d['parity']))"; }
P=29870
run() { N=$1; shift; P=$((P+1)); tag=n${N}_$(echo "$@" | tr ' =' '_-'); [ -z "$1" ] && tag=n${N}_default
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --skip-cpu --e2e-steps 0 > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err; echo "bench N=$N $@ rc=$?"; summ $OUT/bench_$tag.json; }
run 4
run 4 RCV_NO_STAMPS=1
run 4 RCV_BCAST_CTAS=0.25
run 4 RCV_PRE_CTAS=1.0 RCV_BCAST_CTAS=0.25
run 4 RCV_PRE_CTAS=0.85
run 2
run 2 RCV_BCAST_CTAS=0.25
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_hsdp.py tests/test_gpu_realkill.py -q -p no:randomly > $OUT/pytest_dist.log 2>&1; echo "pytest dist rc=$?"; tail -2 $OUT/pytest_dist.log
timeout 600 python tools/sweep.py --n 2,4 --sizes-mb 1,4,16 --reps 7 --out $OUT/sweep_small.jsonl > $OUT/sweep_small.log 2>&1; echo "sweep rc=$?"
python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/r2q/sweep_small.jsonl")]
for r in rows:
    if r["impl"]=="nccl" or (not r["dead"] and r["spares"]==0):
        print("  %-5s n=%d %5d MB %8.1f us busbw %6.1f" % (r["impl"], r["n"], r["bytes"]>>20, r["ms"]*1e3, r.get("busbw_gbs",0)))
PY
