#!/bin/bash
# round-2 job N (4 GPUs): fused drop-in multidev collective (tests + sweep vs
# NCCL, fused vs split), multi-GPU suite at the new defaults (lag 2, 4 sets),
# N=4 trace
OUT=gpurun_out/r2n; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_fold.py -q -k multidevice -p no:randomly > $OUT/pytest_md.log 2>&1; echo "pytest md rc=$?"; tail -2 $OUT/pytest_md.log
timeout 900 python tools/sweep.py --n 2,4 --sizes-mb 1,4,16,64,256,1024 --reps 5 --out $OUT/sweep_4gpu_fused.jsonl > $OUT/sweep_fused.log 2>&1; echo "sweep fused rc=$?"
RCV_MD_SPLIT=1 timeout 900 python tools/sweep.py --n 2,4 --sizes-mb 1,4,16,64 --reps 5 --out $OUT/sweep_4gpu_split.jsonl > $OUT/sweep_split.log 2>&1; echo "sweep split rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/r2n/sweep_4gpu_fused.jsonl", "gpurun_out/r2n/sweep_4gpu_split.jsonl"):
    try: rows=[json.loads(l) for l in open(f)]
    except Exception as e: print(f, e); continue
    print(f)
    for r in rows:
        if r["impl"]=="nccl" or (not r["dead"] and r["spares"]==0):
            print("  %-5s n=%d %5d MB %8.1f us busbw %6.1f" % (r["impl"], r["n"], r["bytes"]>>20, r["ms"]*1e3, r.get("busbw_gbs",0)))
PY
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_hsdp.py tests/test_gpu_realkill.py -q -p no:randomly > $OUT/pytest_dist.log 2>&1; echo "pytest dist rc=$?"; tail -2 $OUT/pytest_dist.log
bash tools/gpu_trace.sh 4 > $OUT/trace_n4.txt 2>&1; echo "trace rc=$?"
