#!/usr/bin/env python
"""BASELINE configs[2]: the gradient-commit sweep — one bucket of 1 MB .. 1 GB
fp32 over n = 2/4/8 replicas with 0-3 dead (highest ids, and a seeded random
choice), through the drop-in ``Communicator.ulfm_allreduce`` (the
reference's call, comm.py:176-201) on CUDA views.

Replicas are placed round-robin over the visible GPUs of this process (one
per GPU when n <= #GPUs; the multi-device kernel reads peers over NVLink).
Times are CUDA events on every involved device (max), after warm-up; inputs
are refreshed from a pristine copy before each timed call so every call
reduces the same data.  algBW = S / t; busBW = 2 (live-1)/live * S / t
(nccl-tests convention).  The reference fold (numpy, one thread, as shipped)
is timed on the same shapes up to --cpu-max-mb.  When every replica has its
own GPU, NCCL's (unmasked) all_reduce over the same device set
(torch.cuda.nccl, single process) is timed at every size in the same file
(impl "nccl").  A case with one live member reduces nothing: it is reported
as a no-op, without bandwidths.  One JSON line per case.
"""

import argparse
import json
import os
import random
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11215_b200.comm import Communicator, ReplicaRole  # noqa: E402


def time_reduce(comm_factory, views, pristine, devices, reps):
    def once():
        for v, p in zip(views.values(), pristine):
            v.copy_(p)
        comm = comm_factory()
        evs = {d: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for d in devices}
        for d in devices:
            evs[d][0].record(torch.cuda.current_stream(d))
        comm.ulfm_allreduce(views)
        for d in devices:
            evs[d][1].record(torch.cuda.current_stream(d))
        for d in devices:
            torch.cuda.synchronize(d)
        return max(a.elapsed_time(z) for a, z in evs.values())
    for _ in range(2):
        once()
    return min(once() for _ in range(reps))


def time_nccl(tensors, devices, reps):
    """torch.cuda.nccl.all_reduce (sum, in place) over one tensor per GPU."""
    import torch.cuda.nccl as nccl

    def once():
        evs = {d: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for d in devices}
        for d in devices:
            evs[d][0].record(torch.cuda.current_stream(d))
        nccl.all_reduce(tensors)
        for d in devices:
            evs[d][1].record(torch.cuda.current_stream(d))
        for d in devices:
            torch.cuda.synchronize(d)
        return max(a.elapsed_time(z) for a, z in evs.values())
    for _ in range(3):
        once()
    return min(once() for _ in range(reps))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="1,4,16,64,256,1024")
    ap.add_argument("--n", default="2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu-max-mb", type=int, default=64)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    n_gpu = torch.cuda.device_count()
    rng = random.Random(1234)
    lines = []
    for n in [int(x) for x in args.n.split(",")]:
        devices = [torch.device("cuda", i % n_gpu) for i in range(n)]
        for mb in [int(x) for x in args.sizes_mb.split(",")]:
            numel = mb * (1 << 20) // 4
            pristine = [torch.randn(numel, generator=torch.Generator().manual_seed(1234 + r)).to(devices[r])
                        for r in range(n)]
            views = {r: torch.empty_like(pristine[r]) for r in range(n)}
            if n <= n_gpu:
                ms = time_nccl([views[r] for r in range(n)], devices, args.reps)
                s = numel * 4
                rec = {"config": "configs[2]", "impl": "nccl", "bytes": s, "n": n, "dead": [],
                       "live": n, "gpus": n, "ms": ms, "algbw_gbs": s / ms / 1e6,
                       "busbw_gbs": 2 * (n - 1) / n * s / ms / 1e6,
                       "note": "unmasked sum, NCCL's own order"}
                print(json.dumps(rec), flush=True)
                lines.append(rec)
            for dead in range(0, min(4, n)):
                for pick in (("highest", list(range(n - dead, n))),
                             ("random", sorted(rng.sample(range(n), dead)))):
                    if dead == 0 and pick[0] == "random":
                        continue
                    live = [r for r in range(n) if r not in pick[1]]
                    for spare in (0, 1):
                        roles = {r: ReplicaRole.MAJOR for r in live}
                        if spare:
                            roles[live[-1]] = ReplicaRole.MAJOR_SPARE
                        lv = {r: views[r] for r in live}
                        ms = time_reduce(lambda: Communicator(live, roles), lv,
                                         [pristine[r] for r in live],
                                         sorted({devices[r] for r in live}, key=lambda d: d.index),
                                         args.reps)
                        s = numel * 4
                        rec = {"config": "configs[2]", "impl": "ours", "bytes": s, "n": n,
                               "dead": pick[1], "dead_pick": pick[0], "live": len(live),
                               "spares": spare, "gpus": len({devices[r].index for r in live}),
                               "ms": ms}
                        if len(live) > 1:
                            rec["algbw_gbs"] = s / ms / 1e6
                            rec["busbw_gbs"] = 2 * (len(live) - 1) / len(live) * s / ms / 1e6
                        else:
                            rec["no_op"] = "one live member: nothing to reduce or send"
                        if mb <= args.cpu_max_mb and spare == 0 and pick[0] == "highest":
                            # the reference's fold as shipped: numpy, one thread
                            arrs = [pristine[r].cpu().numpy() for r in live]
                            t0 = time.perf_counter()
                            total = arrs[0].copy()
                            for a in arrs[1:]:
                                total = total + a
                            for _ in live:
                                _ = total.copy()
                            rec["cpu_reference_ms"] = (time.perf_counter() - t0) * 1e3
                            rec["speedup_vs_cpu"] = rec["cpu_reference_ms"] / ms
                        print(json.dumps(rec), flush=True)
                        lines.append(rec)
            del pristine, views
            torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            for r in lines:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
