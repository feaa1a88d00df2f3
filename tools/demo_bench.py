#!/usr/bin/env python
"""The reference's own CPU demo: W=4 replicas x
G=8 microbatches, K=4 buckets, linear toy model of dim 2^20, replica 1
killed during_sync on bucket 1 at iteration 2, 4 iterations — through the
drop-in run_iteration on the GPU (reference-order fold, fp64, every kernel
ours) and through the CPU oracle (the reference's algorithm in numpy, one
thread, bit-identical accounting).  Prints one JSON line."""

import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11215_b200.metrics import replay_experiment  # noqa: E402
from oracle.protocol import ScriptedKills, World  # noqa: E402

W, G, K, DIM, ITERS = 4, 8, 4, 1 << 20, 4
ENTRIES = [(2, 1, "during_sync:1")]


def main():
    kw = dict(w_init=W, g_init=G, iterations=ITERS, k_buckets=K, dim=DIM,
              model_kind="linear", stream_seed=0, lr=0.05, policy="static")
    replay_experiment(**dict(kw, iterations=1), entries=[])  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows = replay_experiment(**kw, entries=ENTRIES)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    world = World(W, G, k=K, dim=DIM, kind="linear", seed=0, lr=0.05)
    t0 = time.perf_counter()
    cpu_rows = []
    for t in range(ITERS):
        plan = [("during_sync", 1, [1])] if t == 2 else []
        cpu_rows.append(world.iterate(t, ScriptedKills(plan)))
    cpu_s = time.perf_counter() - t0
    same = all(r["contributions"] == sorted([k, v] for k, v in c["contributions"].items())
               and r["events"] == c["events"] for r, c in zip(rows, cpu_rows))
    print(json.dumps({
        "config": "reference CPU demo: W=4 x G=8, K=4, linear dim 2^20, replica 1 killed "
                  "during_sync:1 at iteration 2, 4 iterations",
        "gpu_drop_in_s": gpu_s, "cpu_oracle_s": cpu_s, "speedup": cpu_s / gpu_s,
        "accounting_identical": same,
        "losses_gpu": [r["loss"] for r in rows],
        "losses_cpu": [c["loss"] for c in cpu_rows]}))


if __name__ == "__main__":
    main()
