#!/bin/bash
# round-2 job AI (4 GPUs): cached drop-in argument path: GPU suite, host cost,
# small-bucket sweep vs NCCL
OUT=gpurun_out/r2ai; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > $OUT/pytest_gpu_4gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu_4gpu.txt
timeout 300 python tools/dropin_host.py > $OUT/dropin_host.jsonl 2> $OUT/dropin_host.err; echo "dropin host rc=$?"; cat $OUT/dropin_host.jsonl
timeout 600 python tools/sweep.py --n 2,4 --sizes-mb 1,4,16 --reps 7 --out $OUT/sweep_small.jsonl > $OUT/sweep_small.log 2>&1; echo "sweep rc=$?"
python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/r2ai/sweep_small.jsonl")]
for r in rows:
    if r["impl"]=="nccl" or (not r["dead"] and r["spares"]==0):
        print("  %-5s n=%d %5d MB %8.1f us busbw %6.1f" % (r["impl"], r["n"], r["bytes"]>>20, r["ms"]*1e3, r.get("busbw_gbs",0)))
PY
