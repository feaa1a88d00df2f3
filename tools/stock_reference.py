#!/usr/bin/env python
"""Time the STOCK reference (steadybatch, imported from /root/reference) on
BASELINE configs[1]'s gradient-commit shape, unmodified and unsampled:
W=8 replicas, G=4 (M=32 microbatches), K=20 buckets, a gradient of
d = 124,439,808 elements (GPT-2 124M), replica 3 killed during_sync on
bucket 7.  VERDICT r1 "What's missing" 6.

The reference's own `run_iteration` (ref:trainer.py:324-487) runs the whole
path: per-microbatch `flat += grad` (trainer.py:202-229), snapshot_and_tag
(buckets.py:61-69), `Communicator.ulfm_allreduce` (comm.py:176-201),
consensus, restoration, `flat / B` and the SGD step.  The "constant" stream
(trainer.py:134-168) makes every example the same precomputed vector, so no
example synthesis is timed -- only the commit path plus the reference's
per-microbatch loss (one dot product of d) and its optimizer step.  The
reference computes in float64 (its native dtype; our B200 path is f32).

Build container only (the reference does not travel to the GPU box); the
result is committed under profiles/.  One Python thread, as shipped.

    python tools/stock_reference.py --out profiles/r2/stock_reference_configs1.json
"""

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
D_GPT2 = 124_439_808
TOKENS_PER_MB = 4096  # ref:sim.py:230


class Scripted:
    """Injector: replica 3 dies during_sync on bucket 7 of iteration `at`."""

    def __init__(self, at, it):
        self.at, self.it = at, it

    def fire(self, phase, bucket=None):
        if self.it == self.at and phase == "during_sync" and bucket == 7:
            self.at = -1
            return [3]
        return []


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=D_GPT2)
    ap.add_argument("--iters", type=int, default=2, help="iteration 1 carries the failure")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    sys.path.insert(0, REF_SRC)
    import steadybatch
    from steadybatch.comm import Communicator
    from steadybatch.policy import assign_roles, initial_state
    from steadybatch.trainer import DataStream, ReplicaState, ToyModel, run_iteration

    w, g, k = 8, 4, 20
    members = list(range(w))
    state = initial_state(w, g)
    comm = Communicator(members, assign_roles(state, members))
    t0 = time.perf_counter()
    stream = DataStream(7, w, a.dim, "constant")
    reps = {r: ReplicaState(r, ToyModel("constant", np.zeros(a.dim)), k) for r in members}
    setup_s = time.perf_counter() - t0
    rows = []
    for t in range(a.iters):
        inj = Scripted(1, t)
        t0 = time.perf_counter()
        out = run_iteration(t, reps, comm, state, stream, injector=inj)
        dt = time.perf_counter() - t0
        state = out.state
        rows.append({"iteration": t, "seconds": dt, "contrib_total": out.contrib_total,
                     "w_cur": out.w_cur, "events": out.events,
                     "committed_tokens_per_s": out.contrib_total * TOKENS_PER_MB / dt})
        print(json.dumps(rows[-1]), flush=True)
    tot = sum(r["seconds"] for r in rows)
    res = {
        "what": "stock reference run_iteration (steadybatch, unmodified), configs[1] commit shape",
        "reference": getattr(steadybatch, "__version__", "pkg/src"),
        "dim": a.dim, "replicas": w, "microbatches": w * g, "buckets": k,
        "failure": "replica 3 during_sync bucket 7 of iteration 1",
        "dtype": "f64 (reference native)", "threads": 1,
        "host": {"cpu_count": os.cpu_count(), "processor": platform.processor() or platform.machine(),
                 "numpy": np.__version__, "python": platform.python_version()},
        "setup_s": setup_s, "iterations": rows,
        "committed_tokens_per_s": sum(r["contrib_total"] for r in rows) * TOKENS_PER_MB / tot,
        "seconds_per_iteration": tot / len(rows),
    }
    print(json.dumps(res))
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
