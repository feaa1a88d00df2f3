#!/usr/bin/env python
"""Real-kill recovery benchmark (SURVEY §8(d) "recovery ms", §8(f)2).

configs[1]'s commit (GPT-2 124M gradient, W = 8 replicas x G = 4
microbatches, K = 20 buckets) over `--world` ranks, one process per rank
(ranks share GPUs when the box has fewer).  At step --fail-step rank 1's
process SIGKILLs itself during_sync on bucket --bucket with its kernels in
flight (no drain).  The survivors are not told; they detect, agree, re-form
and recover in-step.  Rank 0 prints one JSON line:

* detect_ms   kill -> the node liveness declares the rank dead (heartbeat
              deadline; CLOCK_MONOTONIC, both stamped in shared memory)
* agree_ms    declared -> the first survivor's poll fixes the failed set
* reform_ms   device time FAILURE -> first recomputed microbatch (the
              protocol's repair and quota decisions, device draining)
* recompute_ms  regenerating the dead replicas' uncommitted microbatch
              gradients on the survivors (stand-in for their backward)
* rereduce_ms   every bucket committed after the recompute
* shrink_ms   torch.distributed.shrink_group (NCCL ranks only), host
* total_ms    detect + agree + device FAILURE -> commit

plus the failure-free / failure / degraded step times and a bitwise check of
every survivor's committed gradient against a torch fp32 canonical tree.

    python tools/realkill_bench.py --world 2 --out gpurun_out/realkill.json
"""

import argparse
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from mp_util import free_port, init_rank  # noqa: E402

W, G, K = 8, 4, 20
VICTIM_RANK = 1


def worker(rank, world, port, q, a):
    try:
        shared = init_rank(rank, world, port)
        from bench import parity_check, recovery_breakdown
        from paper_2605_11215_b200.dist import (DeadPeerDetector, DistributedGradientCommit,
                                                RealKill)
        dev = torch.device("cuda", torch.cuda.current_device())

        def make_leaf(m, out=None):
            gen = torch.Generator(device=dev).manual_seed(1234 + m)
            kw = dict(generator=gen, device=dev, dtype=torch.float32)
            return torch.randn(a.numel, **kw) if out is None else torch.randn(a.numel, out=out, **kw)

        leaves = [make_leaf(m) for m in range(W * G)]
        eng = DistributedGradientCommit(a.numel, W, G, K, real_kill=True,
                                        barrier_timeout_s=a.timeout,
                                        liveness_deadline_s=a.deadline * 1e-3,
                                        liveness_period_s=a.period * 1e-3)
        per = W // world
        victims = set(range(VICTIM_RANK * per, (VICTIM_RANK + 1) * per))
        victim_range = {m for r in victims for m in range(r * G, (r + 1) * G)}
        step = {"t": -1}
        bufs = {m: torch.empty_like(leaves[m]) for m in victim_range}
        regen = {}

        def leaf(m, rid):
            if step["t"] == a.fail_step and m in victim_range and rid not in victims:
                if m not in regen:
                    eng.mark("regen_a")
                    make_leaf(m, out=bufs[m])
                    eng.mark("regen_b")
                    regen[m] = bufs[m]
                return regen[m]
            return leaves[m]

        if rank == VICTIM_RANK:
            inj = RealKill(a.fail_step, "during_sync", a.bucket, liveness=eng.liveness)
        else:
            inj = DeadPeerDetector(eng, shrink=not shared)
        step_ms, outs = [], []
        for t in range(a.fail_step + 1 + a.after):
            step["t"] = t
            inj.step = t
            eng.recovery_events = [] if t == a.fail_step else None
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            out = eng.step(t, leaf, inj)
            s1.record()
            torch.cuda.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            outs.append(out)
            if t == a.fail_step:
                rec = recovery_breakdown(eng)
                eng.recovery_events = None
        mism = parity_check(eng, leaves, a.numel)
        if getattr(inj, "shrinker", None) is not None:
            inj.shrinker.join(timeout=60)
        det = inj.detections[0] if inj.detections else {}
        pre = step_ms[1:a.fail_step]  # step 0 warms up
        res = {
            "metric": "recovery ms after a real rank loss (SIGKILL mid-kernel)",
            "world": world, "shared_gpus": shared, "gpus": torch.cuda.device_count(),
            "numel": a.numel, "replicas": W, "microbatches": W * G, "buckets": K,
            "victim_rank": VICTIM_RANK, "victim_replicas": sorted(victims),
            "killed_at": {"step": a.fail_step, "phase": "during_sync", "bucket": a.bucket},
            "detected_at": {k: det.get(k) for k in ("phase", "bucket", "poll")},
            "liveness": {"period_ms": a.period, "deadline_ms": a.deadline},
            "detect_ms": det.get("detect_ms"), "agree_ms": det.get("agree_ms"),
            "shrink_ms": det.get("shrink_ms"), "shrink_error": det.get("shrink_error"),
            "reform_host_ms": outs[a.fail_step].reform_host_s * 1e3,
            "device": rec,
            "step_ms": {"failure_free_median": statistics.median(pre) if pre else None,
                        "failure_step": step_ms[a.fail_step],
                        "degraded_median": statistics.median(step_ms[a.fail_step + 1:])
                        if a.after else None,
                        "all": [round(x, 3) for x in step_ms]},
            "contrib_total": [o.contrib_total for o in outs],
            "w_cur": [o.w_cur for o in outs],
            "events": outs[a.fail_step].events,
            "parity": "bitwise" if mism == 0 else "fail", "mismatched_elements": mism,
            "integrity_errors_during_recovery": eng.integrity_errors,
        }
        if rec and det.get("detect_ms") is not None:
            res["total_ms"] = det["detect_ms"] + (det.get("agree_ms") or 0.0) + rec["total_ms"]
        q.put((rank, res))
    except Exception:
        import traceback
        q.put((rank, "ERROR\n" + traceback.format_exc()))
    q.close()
    q.join_thread()
    os._exit(0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--numel", type=int, default=124_439_808)
    ap.add_argument("--fail-step", type=int, default=4)
    ap.add_argument("--after", type=int, default=3)
    ap.add_argument("--bucket", type=int, default=7)
    ap.add_argument("--deadline", type=float, default=10.0, help="liveness deadline, ms")
    ap.add_argument("--period", type=float, default=1.0, help="heartbeat period, ms")
    ap.add_argument("--timeout", type=float, default=30.0, help="barrier timeout, s")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    port = free_port()
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, a.world, port, q, a)) for r in range(a.world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(a.world - 1):
        r, res = q.get(timeout=900)
        got[r] = res
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    errs = {r: v for r, v in got.items() if isinstance(v, str)}
    if errs:
        print(json.dumps({"failed": errs}))
        sys.exit(1)
    line = dict(got[0])
    line["victim_exitcode"] = procs[VICTIM_RANK].exitcode
    line["survivors_agree"] = len({json.dumps(v["detected_at"]) for v in got.values()}) == 1
    line["survivor_parity"] = {r: v["parity"] for r, v in got.items()}
    print(json.dumps(line))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(line, f, indent=1)
    ok = all(v["parity"] == "bitwise" for v in got.values()) and line["survivors_agree"]
    sys.exit(0 if ok else 2)


if __name__ == "__main__":
    main()
