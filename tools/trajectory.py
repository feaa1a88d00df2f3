#!/usr/bin/env python
"""BASELINE configs[4] (and configs[0]): train the tiny transformer for
`--steps` optimizer steps through the canonical executor, once failure-free
and once under successive replica failures (8 -> 4), and compare the loss
and parameter trajectories.  Prints one JSON summary line; `--out` also
writes per-step losses.

Replicas are simulated on one GPU (the reference's single-process model);
the data of step t's microbatch m is a pure function of (t, m).  The claim
checked here is the north star's: the loss trajectory under failures
matches the failure-free run — bit for bit, because the canonical commit's
result depends only on the microbatch gradients, and survivors recompute
exactly the dead replica's uncommitted microbatches.
"""

import argparse
import json
import os
import sys
import time

os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11215_b200.executor import (CanonicalExecutor, TinyTransformer,  # noqa: E402
                                            lm_loss, synthetic_lm_batch)

# successive failures 8 -> 4 (the survey's seeded example steps 11, 335,
# 402, 403; one victim per failure, all three injection locations)
SCHEDULE = {11: [("during_sync", 1, [2])], 335: [("after_sync", None, [5])],
            402: [("before_sync", None, [0])], 403: [("during_sync", 0, [7])]}


class Schedule:
    def __init__(self, plan):
        self.plan = {t: list(v) for t, v in plan.items()}
        self.t = -1

    def fire(self, phase, bucket=None):
        cur = self.plan.get(self.t, [])
        hit = [e for e in cur if e[0] == phase and (phase != "during_sync" or e[1] == bucket)]
        self.plan[self.t] = [e for e in cur if e not in hit]
        return [r for e in hit for r in e[2]]


def run(args, plan):
    torch.use_deterministic_algorithms(True)
    torch.manual_seed(args.seed)
    model = TinyTransformer(layers=args.layers, d=args.d, heads=4, seq=args.seq)
    ex = CanonicalExecutor(model, synthetic_lm_batch(args.seed, micro=args.micro, seq=args.seq),
                           lm_loss, args.w, args.g, args.k, lr=args.lr)
    sched = Schedule(plan)
    losses, step_ms, events = [], [], []
    for t in range(args.steps):
        sched.t = t
        a = torch.cuda.Event(enable_timing=True)
        z = torch.cuda.Event(enable_timing=True)
        a.record()
        out, loss = ex.step(t, sched)
        z.record()
        torch.cuda.synchronize()
        step_ms.append(a.elapsed_time(z))
        losses.append(loss)
        if out.events:
            events.append({"step": t, "w_cur": out.w_cur, "events": out.events,
                           "recomputed": len([c for c in ex.computed if c[0] == t]) - args.w * args.g})
        assert out.contrib_total == args.w * args.g
    return losses, ex.flat.clone(), step_ms, events, ex.numel


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--w", type=int, default=8)
    ap.add_argument("--g", type=int, default=4)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--seq", type=int, default=64)
    ap.add_argument("--micro", type=int, default=4)
    ap.add_argument("--lr", type=float, default=0.1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    plan = {t: v for t, v in SCHEDULE.items() if t < args.steps}
    t0 = time.time()
    ref_l, ref_p, ref_ms, _, numel = run(args, {})
    l, p, ms, events, _ = run(args, plan)
    same_losses = ref_l == l
    first_diff = next((t for t, (a, b) in enumerate(zip(ref_l, l)) if a != b), None)
    summary = {
        "config": "configs[4]: successive failures %d->%d over %d steps, tiny transformer "
                  "(%d params), M=%d" % (args.w, args.w - len(plan), args.steps, numel,
                                          args.w * args.g),
        "loss_trajectory_bitwise_equal": same_losses,
        "params_bitwise_equal": bool(torch.equal(ref_p, p)),
        "first_differing_step": first_diff,
        "loss_first_last": [ref_l[0], ref_l[-1]],
        "failures": events,
        "step_ms_median_failure_free_run": sorted(ref_ms)[len(ref_ms) // 2],
        "step_ms_median_failure_run": sorted(ms)[len(ms) // 2],
        "failure_step_ms": {e["step"]: ms[e["step"]] for e in events},
        "wall_s": time.time() - t0,
    }
    print(json.dumps(summary))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(dict(summary, losses_failure_free=ref_l, losses_with_failures=l), f)


if __name__ == "__main__":
    main()
