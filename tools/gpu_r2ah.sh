#!/bin/bash
# round-2 job AH (1 GPU): pipelined e2e copies (two H2D streams, overlapped
# D2H) at N=1
OUT=gpurun_out/r2ah; mkdir -p $OUT
for rep in 1 2; do
timeout 600 python bench.py --skip-cpu --e2e-steps 6 > $OUT/bench_n1_$rep.json 2> $OUT/bench_n1_$rep.err; echo "bench N=1 rc=$?"
python -c "
import json; d=json.loads(open('$OUT/bench_n1_$rep.json').read().strip().splitlines()[-1]); print(d['value']/1e6, d['parity'], d['e2e'])"
done
