#!/usr/bin/env python
"""Repeat the whole-rank-death scenarios of tests/test_gpu_dist.py many
times inside one multi-process job and log every trial (bitwise result per
bucket, stamp/timeout status words).

    python tools/repeat_dist.py --world 8 --trials 100 --out gpurun_out/rep8.jsonl

One replica per rank, W = world, G = 4, K = 20 (configs[1]'s shape at
world = 8), a fresh engine per trial, the victim and its bucket drawn from a
seeded RNG; sizes alternate between a tiny and a multi-MB gradient so both
short and long kernels race.  Ranks share the box's GPUs round-robin when
world exceeds the device count (gloo handshakes)."""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from mp_util import failed, spawn  # noqa: E402


class Kill:
    def __init__(self, plan):
        self.plan = list(plan)

    def fire(self, phase, bucket=None):
        hit = [e for e in self.plan if e[0] == phase and (phase != "during_sync" or e[1] == bucket)]
        self.plan = [e for e in self.plan if e not in hit]
        return [r for e in hit for r in e[2]]


def worker(rank, world, trials, seed, sizes):
    from paper_2605_11215_b200.dist import CommitIntegrityError, DistributedGradientCommit
    from oracle import fold
    g, k = 4, 20
    b = world * g
    rng = np.random.default_rng(seed)
    data = {}
    for numel in sizes:
        host = [np.random.default_rng(700 + m).standard_normal(numel).astype(np.float32)
                for m in range(b)]
        data[numel] = ([torch.from_numpy(h).cuda() for h in host],
                       fold.canonical_tree(dict(enumerate(host)), b) / np.float32(b))
    out = []
    for t in range(trials):
        numel = sizes[t % len(sizes)]
        dev, want = data[numel]
        victim = int(rng.integers(0, world))
        bucket = int(rng.integers(0, k))
        phase = ("during_sync", "during_sync", "after_sync", "before_sync")[int(rng.integers(0, 4))]
        plans = [[], [(phase, bucket if phase == "during_sync" else None, [victim])], []]
        eng = DistributedGradientCommit(numel, world, g, k, barrier_timeout_s=60.0)
        bad_steps, err = [], None
        t0 = time.perf_counter()
        for s, plan in enumerate(plans):
            # a step that raised has still run to its end on every rank:
            # record the error and keep the ranks in lockstep
            try:
                eng.step(s, lambda m, rid: dev[m], Kill(plan))
            except CommitIntegrityError as exc:
                err = err or str(exc)
            torch.cuda.synchronize()
            bad = set()
            for r in eng.comm.members:
                if eng._holds(r):
                    got = eng.grads[r].cpu().numpy()
                    bad |= {j for j, (lo, hi) in enumerate(eng.bounds)
                            if got[lo:hi].tobytes() != want[lo:hi].tobytes()}
            bad_steps.append(sorted(bad))
        try:
            eng.check_peers()
        except CommitIntegrityError as exc:
            err = err or str(exc)
        out.append(dict(trial=t, numel=numel, victim=victim, phase=phase, bucket=bucket,
                        bad=bad_steps, status=eng.status.tolist(), error=err,
                        ms=(time.perf_counter() - t0) * 1e3))
        eng.rt.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--trials", type=int, default=100)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--sizes", default="6464,2560064")
    ap.add_argument("--out", default="gpurun_out/repeat.jsonl")
    a = ap.parse_args()
    sizes = [int(x) for x in a.sizes.split(",")]
    t0 = time.time()
    res = spawn(worker, a.world, a.trials, a.seed, sizes, timeout=3600)
    if failed(res):
        print(json.dumps({"failed": failed(res)}))
        sys.exit(1)
    n_bad = n_err = 0
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        for t in range(a.trials):
            rows = [res[r][t] for r in range(a.world)]
            bad = any(any(s) for row in rows for s in row["bad"])
            err = any(row["error"] for row in rows)
            n_bad += bad
            n_err += err
            f.write(json.dumps({"trial": t, "bitwise": not bad, "integrity_error": err,
                                "env_reuse": os.environ.get("RCV_REUSE", "1"),
                                "ranks": rows}) + "\n")
    summary = {"world": a.world, "trials": a.trials, "bitwise_trials": a.trials - n_bad,
               "integrity_errors": n_err, "gpus": torch.cuda.device_count(),
               "reuse": os.environ.get("RCV_REUSE", "1"), "sizes": sizes,
               "wall_s": time.time() - t0}
    print(json.dumps(summary))
    sys.exit(0 if n_bad == 0 and n_err == 0 else 2)


if __name__ == "__main__":
    main()
