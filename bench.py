#!/usr/bin/env python
"""Benchmark of the ReCoVer data-parallel gradient commit on B200.

Workload (BASELINE.json configs[1]): the GPT-2 124M gradient
(d = 124,439,808 fp32 = 497.8 MB), DP = 8 replicas, M = 32 microbatches per
optimizer step (G = 4 per replica), K = 20 buckets (~25 MB), replica 3 killed
``during_sync`` on bucket 7 in the middle of the timed region.  At N=1 the
eight replicas live on one GPU (the reference's own single-process model).

A "step" is one optimizer step's gradient commit: the fused canonical-order
accumulate + survivor-masked reduce + 1/M scale of all 32 microbatch
gradients (synthetic, resident in HBM; they stand for the backward outputs)
into every live replica's gradient buffer, through GradientCommit.step with
the failure schedule, recovery included.

Metric: committed tokens/s (tokens_per_microbatch = 4096, sim.py:230) under
the failure schedule; the line also carries the commit kernel's HBM GB/s vs
the measured peak (roofline) and recovery ms.  ``--impl reference`` times the
reference algorithm (the oracle port of comm.py/trainer.py: per-replica
`flat += grad`, snapshot copies, ascending masked fold, rewinds) on the host
cores over a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D_GPT2 = 124_439_808
W, G, K = 8, 4, 20
M = W * G
TOKENS_PER_MB = 4096
VICTIM, VICTIM_BUCKET = 3, 7
METRIC = "committed tokens/s under failure schedule; masked-allreduce GB/s; recovery ms"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--numel", type=int, default=D_GPT2)
    ap.add_argument("--buckets", type=int, default=K)
    ap.add_argument("--no-fail", action="store_true")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--combine-variant", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--cpu-sample", type=int, default=1 << 23)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--trace", default="", help="torch.profiler chrome trace prefix (diagnostics)")
    ap.add_argument("--trace-degraded", action="store_true",
                    help="with --trace: kill the victim in warmup step 0, trace the degraded layout")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """SM clock and clock-event reasons sampled in-process through NVML every
    ~2 ms while the timed region runs (the region is tens of ms, too short
    for `nvidia-smi -lms`).  Reports the median SM clock under load."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.err = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception as exc:  # no NVML: report unsampled
            self.err = repr(exc)
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception as exc:
                self.err = repr(exc)
                return
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if getattr(self, "thread", None):
            self.thread.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"],
                    "error": self.err}
        reasons = sorted({name for _, rs in self.samples for name, attr in self.REASONS
                          if rs & getattr(self.nv, attr, 0)})
        return {"sm_mhz": statistics.median(sm for sm, _ in self.samples),
                "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml"}


class StepKill:
    """Kill VICTIM during_sync on VICTIM_BUCKET at one step (configs[1])."""

    def __init__(self, at_step, bucket=VICTIM_BUCKET):
        self.at_step = at_step
        self.bucket = bucket
        self.step = -1

    def fire(self, phase, bucket=None):
        if self.step == self.at_step and phase == "during_sync" and bucket == self.bucket:
            return [VICTIM]
        return []


# ---------------------------------------------------------------------------
# CPU legs: the reference algorithm (oracle port) on a bounded sample

def _threads():
    return max(1, os.cpu_count() or 1)


def _chunked(n, fn):
    """Run fn(lo, hi) over n elements split across all host threads (numpy
    releases the GIL inside ufuncs)."""
    nt = _threads()
    edges = [n * i // nt for i in range(nt + 1)]
    ths = [threading.Thread(target=fn, args=(edges[i], edges[i + 1])) for i in range(nt)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return nt


def reference_step_sample(leaves, fail_bucket=None):
    """One optimizer step of the reference's data path on a sample:
    trainer.py:192,212 (zero + `flat += grad` per round), buckets.py:68
    (snapshot copies), comm.py:191-200 (ascending fold, write all members),
    on failure buckets.py:136 (rewinds) and the extension pass, then
    trainer.py:446 (`flat / B`)."""
    import numpy as np
    from oracle import fold
    n = leaves[0].shape[0]
    kb = K
    bounds = [(i * (n // kb), n if i == kb - 1 else (i + 1) * (n // kb)) for i in range(kb)]
    flats = [np.zeros(n, dtype=np.float32) for _ in range(W)]
    snaps = [np.empty(n, dtype=np.float32) for _ in range(W)]

    def run(lo, hi):
        for r in range(W):
            for j in range(G):
                flats[r][lo:hi] += leaves[r * G + j][lo:hi]
        members = list(range(W))

        def cascade(ks, mem):
            for k in ks:
                a, b = bounds[k]
                a, b = max(a, lo), min(b, hi)
                if a >= b:
                    continue
                for r in mem:
                    snaps[r][a:b] = flats[r][a:b]
                tot = fold.masked_fold([flats[r][a:b] for r in mem], [True] * len(mem))
                for r in mem:
                    flats[r][a:b] = tot
        if fail_bucket is None:
            cascade(range(kb), members)
        else:
            cascade(range(fail_bucket), members)
            members = [r for r in members if r != VICTIM]
            for k in range(fail_bucket + 1):          # rewind stale buckets
                a, b = bounds[k]
                a, b = max(a, lo), min(b, hi)
                for r in members:
                    if a < b:
                        flats[r][a:b] = snaps[r][a:b]
            for r in members[:4]:                      # g_ext=1, 3 boundary minors
                flats[r][lo:hi] += leaves[VICTIM * G + members.index(r)][lo:hi]
            cascade(range(kb), members)
        upd = flats[members[0]][lo:hi] / np.float32(M)
        del upd

    return _chunked(n, run)


def cpu_leg(sample, steps, fail_index, warmup=1):
    """Time the reference algorithm on `sample` elements per step; scale to
    the full gradient.  Returns (tokens/s, seconds per full step, threads)."""
    import numpy as np
    rng = np.random.default_rng(1234)
    leaves = [rng.standard_normal(sample, dtype=np.float32) for _ in range(M)]
    for _ in range(max(1, warmup)):
        reference_step_sample(leaves)  # warm caches / page in
    t0 = time.perf_counter()
    nt = 1
    for s in range(steps):
        nt = reference_step_sample(leaves, VICTIM_BUCKET if s == fail_index else None)
    dt = time.perf_counter() - t0
    per_full = dt / steps * (D_GPT2 / sample)
    return M * TOKENS_PER_MB / per_full, per_full, nt


def config_dict(args, world):
    """The workload as both arms report it (identical dicts)."""
    return {"workload": "gpt2-124m gradient commit, DP=8, M=32, K=%d, replica 3 killed "
                        "during_sync:%d" % (args.buckets, min(VICTIM_BUCKET, args.buckets - 1)),
            "numel": args.numel, "replicas": W, "microbatches": M, "buckets": args.buckets,
            "tokens_per_microbatch": TOKENS_PER_MB,
            "fail_step": -1 if args.no_fail else args.warmup + args.steps // 2,
            "placement": "8 replicas on 1 GPU" if world == 1
            else "%d replicas per rank, NVLink P2P" % (W // world),
            "l2": "inputs 15.9 GB >> 126 MB L2 (no flush needed)",
            "parallelism": "dp8-sim" if world == 1 else "dp8 over %d ranks" % world}


def run_reference_arm(args):
    """The reference's CPU data path (oracle port, all host threads) on a
    bounded sample per step: --warmup untimed steps, then --steps timed
    ones, the middle one with the failure.  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    fail = -1 if args.no_fail else args.steps // 2
    tps, per_full, nt = cpu_leg(args.cpu_sample, args.steps, fail, warmup=args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": tps, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_full * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args, world),
        "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": nt, "kind": "port",
                         "sample": "%d of %d elements per step (every microbatch gradient, "
                                   "snapshot, fold and rewind of the reference path on that "
                                   "slice), %d timed steps, scaled linearly to the full gradient"
                                   % (args.cpu_sample, D_GPT2, args.steps)},
        "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# GPU arm

def _lib_launches():
    from paper_2605_11215_b200 import _lib
    return _lib.launch_count()


def torch_reference_tree(leaves, lo, hi, b):
    """The canonical dyadic tree of leaves[lo:hi] (all b present, b a power
    of two) divided by b, evaluated with plain torch fp32 ops: IEEE
    round-to-nearest adds level by level and a true division; independent of
    librcv (the bench's parity check)."""
    vals = [t[lo:hi] for t in leaves]
    while len(vals) > 1:
        vals = [vals[i] + vals[i + 1] for i in range(0, len(vals), 2)]
    return vals[0] / float(b)


def parity_check(eng, leaves, numel, chunk=1 << 24):
    """Bitwise comparison of every live replica this rank holds against the
    torch reference tree; returns the number of mismatching elements."""
    import torch
    mine = [r for r in eng.comm.members if r in eng.grads]
    bad = 0
    for lo in range(0, numel, chunk):
        hi = min(numel, lo + chunk)
        want = torch_reference_tree(leaves, lo, hi, M)
        for r in mine:
            bad += int((eng.grads[r][lo:hi].view(torch.int32) != want.view(torch.int32)).sum())
    return bad


def recovery_breakdown(eng):
    """Device-time split of the failure step from the engine's recovery
    marks: FAILURE -> first recomputed microbatch (the protocol's repair
    and quota decisions on the host, device still draining the first pass),
    recompute (regenerating the dead replica's uncommitted microbatch
    gradients on the survivors), re-reduce (every bucket committed after the
    recompute, the step's closing barrier included).  The parts sum to the
    total, FAILURE -> commit."""
    ev = eng.recovery_events or []
    names = [n for n, _, _ in ev]
    if "fail" not in names or "commit" not in names:
        return None
    fail = ev[names.index("fail")]
    commit = ev[len(names) - 1 - names[::-1].index("commit")]
    regen = [(a, z) for (na, a, _), (nz, z, _) in zip(ev, ev[1:]) if na == "regen_a" and nz == "regen_b"]
    total = fail[1].elapsed_time(commit[1])
    if regen:
        first, last = regen[0][0], regen[-1][1]
        reform = fail[1].elapsed_time(first)
        recompute = sum(a.elapsed_time(z) for a, z in regen)
        gaps = first.elapsed_time(last) - recompute
        rereduce = last.elapsed_time(commit[1]) + gaps
    else:
        reform, recompute, rereduce = 0.0, 0.0, total
    return {"total_ms": total, "detect_ms": 0.0, "reform_ms": reform,
            "recompute_ms": recompute, "rereduce_ms": rereduce,
            "recomputed_microbatches": len(regen),
            "reform_host_ms": None, "detect_note": "simulated kill: the injector reports the "
            "death at the collective (real detection: tools/realkill_bench.py)"}


def run_ours(args):
    import torch
    from paper_2605_11215_b200.commit import GradientCommit

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numel = args.numel

    # synthetic per-microbatch gradients (the backward outputs), resident in
    # HBM.  Microbatch m's gradient is a function of m alone (its own seeded
    # generator), so a survivor that recomputes it gets the same bits.
    def make_leaf(m, out=None):
        gen = torch.Generator(device=dev).manual_seed(1234 + m)
        if out is None:
            return torch.randn(numel, generator=gen, device=dev, dtype=torch.float32)
        return torch.randn(numel, generator=gen, device=dev, dtype=torch.float32, out=out)

    leaves = [make_leaf(m) for m in range(M)]
    total_steps = args.warmup + args.steps
    fail_step = -1 if args.no_fail else args.warmup + args.steps // 2
    if args.trace and args.trace_degraded:
        fail_step = 0
    if world > 1:
        from paper_2605_11215_b200.dist import DistributedGradientCommit
        eng = DistributedGradientCommit(numel, W, G, args.buckets, variant=args.variant,
                                        combine_variant=args.combine_variant)
    else:
        eng = GradientCommit(numel, W, G, args.buckets, placement={r: dev for r in range(W)},
                             variant=args.variant)
    kill = StepKill(fail_step, min(VICTIM_BUCKET, args.buckets - 1))

    # the failure step charges real work for the microbatches the dead
    # replica had not committed: a survivor that takes one over regenerates
    # its gradient on the device (standing in for that microbatch's
    # backward), bracketed by recovery marks
    victim_range = set(range(VICTIM * G, (VICTIM + 1) * G))
    # the recompute's output buffers exist before the step, as backward's
    # would in a training loop (no allocation inside the timed region)
    regen_bufs = {m: torch.empty_like(leaves[m]) for m in victim_range}
    regen_done = {}

    def leaf(m, rid):
        if kill.step == kill.at_step and m in victim_range and rid != VICTIM:
            if regen_done.get(m) != kill.step:
                buf = regen_bufs[m]
                eng.mark("regen_a")
                make_leaf(m, out=buf)
                eng.mark("regen_b")
                regen_done[m] = kill.step
            return regen_bufs[m]
        return leaves[m]

    stream = torch.cuda.current_stream(dev)
    step_ev = []
    outcomes = []
    for s in range(args.warmup):
        kill.step = s
        eng.step(s, leaf, kill)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    if args.trace:
        # diagnostics only: a CUPTI timeline of a few steps, then exit
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            for s in range(args.warmup, args.warmup + 4):
                kill.step = -1
                eng.step(s, leaf, kill)
            torch.cuda.synchronize()
        prof.export_chrome_trace("%s_rank%d.json" % (args.trace, rank))
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    # per-kernel pass: a few failure-free steps with CUDA events around every
    # launch (events between launches perturb cross-stream overlap, so the
    # headline region below runs without them)
    kill.step = -1
    eng.start_timing()
    for s in range(3):
        eng.step(args.warmup + s, leaf, None)
    torch.cuda.synchronize()
    recs = eng.drain_timing()
    if world > 1:
        torch.distributed.barrier()
    eng.recovery_events = []
    n_launch0 = _lib_launches()
    with Clocks(local) as clk:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        # every rank enters the timed region together (the clock sampler's
        # start-up differs per rank, and the max over ranks would otherwise
        # count one rank's wait for the slowest one's first barrier)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()
        start.record(stream)
        t_host = time.perf_counter()
        host_step = []
        prof0 = dict(getattr(eng, "host_prof", {}))
        for s in range(args.warmup, total_steps):
            kill.step = s
            a = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            h0 = time.perf_counter()
            outcomes.append(eng.step(s, leaf, kill))
            host_step.append((time.perf_counter() - h0) * 1e3)
            step_ev.append(a)
        end.record(stream)
        host_ms = (time.perf_counter() - t_host) * 1e3 / args.steps
        torch.cuda.synchronize()
    n_launch = _lib_launches() - n_launch0
    elapsed_ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    step_ev.append(end)
    step_ms = [step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(len(step_ev) - 1)]
    committed = sum(o.contrib_total for o in outcomes)
    tokens = committed * TOKENS_PER_MB
    value = tokens / (elapsed_ms / 1e3)
    # the paper's effective throughput: processed tokens /
    # (runtime x alive GPUs), each step weighted by the GPUs still holding a
    # live replica at its end
    per = W // world
    gpu_s = sum(ms / 1e3 * len({rid // per for rid in o.contributions})
                for ms, o in zip(step_ms, outcomes))
    fail_idx = [i for i, o in enumerate(outcomes) if o.events]
    recovery = recovery_breakdown(eng) if fail_idx else None
    if recovery is not None:
        recovery["reform_host_ms"] = outcomes[fail_idx[0]].reform_host_s * 1e3
    eng.recovery_events = None

    # the bench proves its own number: after the timed region every live
    # replica's committed gradient (the last step's, degraded layout when a
    # replica died) must equal the canonical tree evaluated independently
    # with plain torch ops, bit for bit
    mism = parity_check(eng, leaves, numel)
    if world > 1:
        t = torch.tensor([mism], device=dev, dtype=torch.int64)
        torch.distributed.all_reduce(t)
        mism = int(t.item())

    # the same per-kernel pass over 2 steps of the degraded layout (after the
    # timed region, so the headline is unperturbed)
    recs_deg = []
    if fail_step >= 0:
        eng.start_timing()
        for s in range(2):
            eng.step(total_steps + s, leaf, None)
        torch.cuda.synchronize()
        recs_deg = eng.drain_timing()
        if world > 1:
            torch.distributed.barrier()

    kinds, per_kind = summarise_kernels(recs)
    per_kind_deg = summarise_kernels(recs_deg)[1]
    peak, peak_kind = peaks()
    dom = max(kinds, key=lambda kk: kinds[kk]["ms"]) if kinds else None
    # the failure step against the failure-free steps before it (the steps
    # after it run the degraded layout, reported separately)
    pre = step_ms[:fail_idx[0]] if fail_idx else step_ms
    post = step_ms[fail_idx[-1] + 1:] if fail_idx else []
    if recovery is not None and pre:
        recovery["failure_step_extra_ms"] = step_ms[fail_idx[0]] - statistics.median(pre)

    # e2e through the public API with host buffers: pinned host gradients
    # copied in every step, committed gradient copied out every step
    e2e = None
    if args.e2e_steps > 0:
        e2e = e2e_leg(args, dev, leaves, numel, world)
    if world > 1:
        eng.check_peers()

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": config_dict(args, world),
        "parity": "bitwise" if mism == 0 else "fail",
        "parity_detail": {"mismatched_elements": mism, "checked": "every live replica's "
                          "committed gradient after the timed region vs a torch fp32 "
                          "canonical tree / B over all %d microbatch gradients" % M},
        "roofline": roofline(dom, per_kind, peak, peak_kind, world),
        "kernels": per_kind,
        "kernels_degraded": per_kind_deg or None,
        # masked-allreduce algorithmic bandwidth: gradient bytes committed
        # (reduced over the live replicas and scaled) per second of step time
        "allreduce_algbw_gbs": numel * 4 / (elapsed_ms / args.steps / 1e3) / 1e9,
        "effective_tokens_per_s_per_alive_gpu": tokens / gpu_s if gpu_s else None,
        "recovery_ms": recovery["total_ms"] if recovery else None,
        "recovery": recovery,
        "step_ms": {"median": statistics.median(step_ms), "max": max(step_ms),
                    "failure_step": step_ms[fail_idx[0]] if fail_idx else None,
                    "failure_free_median": statistics.median(pre) if pre else None,
                    "degraded_median": statistics.median(post) if post else None,
                    "all": [round(x, 3) for x in step_ms]},
        "host_enqueue_ms_per_step": host_ms,
        # where the host time goes (multi-process engine): plan lookup/build,
        # the native per-bucket enqueue, the wait for the previous step's
        # status words (the GPU running behind the host)
        "host_prof_ms_per_step": {k: (v - prof0.get(k, 0.0)) * 1e3 / args.steps
                                  for k, v in getattr(eng, "host_prof", {}).items()} or None,
        # host time inside eng.step (control plane + launches): a step whose
        # host time exceeds its device time leaves the GPU waiting
        "host_step_ms": {"failure_free_median": statistics.median(host_step[:fail_idx[0]])
                         if fail_idx and fail_idx[0] > 0 else statistics.median(host_step),
                         "degraded_median": statistics.median(host_step[fail_idx[-1] + 1:])
                         if fail_idx and fail_idx[-1] + 1 < len(host_step) else None},
        "gpu_launches": n_launch,
        "kernel_pass": "per-kernel rows from 3 failure-free steps timed launch by launch (CUDA events on each launch's stream) before the headline region",
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if rank == 0 and not args.skip_cpu:
        tps, per_full, nt = cpu_leg(args.cpu_sample, 2, 1)
        line["cpu_baseline"] = {"value": tps, "unit": "tokens/s", "cores": nt, "kind": "port",
                                "sample": "%d of %d elements per step, 2 steps (one with "
                                          "the failure), scaled linearly" % (args.cpu_sample, D_GPT2)}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    if mism:
        sys.exit(3)


NVLINK_PEAK = 770.0  # GB/s per direction, measured peer copy (B200_PROFILING.md)
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def traffic_of(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed ncu --set full capture of this build
    (profiles/ncu_traffic.json, written by tools/ncu_summarize.py traffic),
    or None when no capture of that kernel is committed."""
    try:
        with open(TRAFFIC_FILE) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    row = d.get("kernels", {}).get(kernel)
    return None if row is None else row.get("dram_bytes")


def summarise_kernels(recs):
    """Per kernel kind: launches, mean launch time, HBM and NVLink rates
    (CUDA events on the launching stream around every launch)."""
    kinds = {}
    for kind, ms, nb, nin, nout in recs:
        k = kinds.setdefault(kind, {"launches": 0, "ms": 0.0, "bytes": 0, "nvl_in": 0, "nvl_out": 0})
        k["launches"] += 1
        k["ms"] += ms
        k["bytes"] += nb
        k["nvl_in"] += nin
        k["nvl_out"] += nout
    per_kind = {}
    for kind, k in kinds.items():
        sec = k["ms"] / 1e3
        # NVLink per direction: this rank's remote reads arrive inbound while
        # the peers' reads of its slices leave outbound (and its remote
        # stores leave while the peers' arrive), so with symmetric traffic
        # each direction carries remote reads + remote writes
        per_kind[kind] = {
            "launches": k["launches"], "mean_launch_us": 1e3 * k["ms"] / k["launches"],
            "hbm_gbs": k["bytes"] / sec / 1e9 if sec else None,
            "nvlink_gbs_per_direction": (k["nvl_in"] + k["nvl_out"]) / sec / 1e9 if sec else None}
    return kinds, per_kind


def roofline(dom, per_kind, peak, peak_kind, world=1):
    if dom is None:
        return None
    k = per_kind[dom]
    if dom == "combine" and (k["nvlink_gbs_per_direction"] or 0) > 0:
        ach = k["nvlink_gbs_per_direction"]
        # the per-kernel pass runs failure-free steps: one cover node per
        # rank, a perfect tree of world leaves, which AUTO runs DIRECT
        return {"bound": "nvlink", "achieved": ach, "peak": NVLINK_PEAK, "unit": "GB/s",
                "frac": ach / NVLINK_PEAK, "traffic": None, "peak_kind": "measured peer copy",
                "kernel": "fold_direct_pair_kernel<ProgFull<%d>> combine over peer pointers "
                          "(failure-free cover; degraded covers run the fixed programs of "
                          "shapes.inc, see kernels_degraded)" % max(0, world.bit_length() - 1),
                "mean_launch_us": k["mean_launch_us"], "launches_timed": k["launches"],
                "hbm_gbs": k["hbm_gbs"]}
    # the accumulator type the library picks for the N=1 commit's perfect
    # tree (librcv's RCV_W256: 2 = 256-bit vectors with streaming stores)
    acc = {"0": "float", "1": "F8W"}.get(os.environ.get("RCV_W256", "2"), "F8WS")
    name = "fold_direct_kernel<%s, ProgFull<5>>" % acc
    return {"bound": "hbm", "achieved": k["hbm_gbs"], "peak": peak, "unit": "GB/s",
            "frac": k["hbm_gbs"] / peak if k["hbm_gbs"] else None,
            "traffic": traffic_of(name), "peak_kind": peak_kind,
            "kernel": "%s (rcv_tree_commit AUTO, %s)" % (name, dom),
            "mean_launch_us": k["mean_launch_us"], "launches_timed": k["launches"]}


def e2e_leg(args, dev, leaves, numel, world=1):
    """The same step through the public API with HOST inputs: every step each
    rank copies its replicas' microbatch gradients host->device (pinned) and
    its committed gradient device->host, inside the timed region (max over
    ranks).  Under the same failure schedule as the headline: replica 3 dies
    during_sync on bucket 7 of the middle timed step (a fresh engine)."""
    import torch
    from paper_2605_11215_b200.commit import GradientCommit
    if world > 1:
        from paper_2605_11215_b200.dist import DistributedGradientCommit
        eng = DistributedGradientCommit(numel, W, G, args.buckets, variant=args.variant,
                                        combine_variant=args.combine_variant)
    else:
        eng = GradientCommit(numel, W, G, args.buckets, placement={r: dev for r in range(W)},
                             variant=args.variant)
    mine = [r for r in range(W) if r in eng.grads]
    idx = [m for r in mine for m in range(r * G, (r + 1) * G)]  # failure-free canonical ranges
    try:
        host = {m: torch.empty(numel, dtype=torch.float32, pin_memory=True) for m in idx}
        pinned = True
    except RuntimeError:
        host = {m: torch.empty(numel, dtype=torch.float32) for m in idx}
        pinned = False
    for m in idx:
        host[m].copy_(leaves[m])
    out_host = torch.empty(numel, dtype=torch.float32, pin_memory=pinned)
    stream = torch.cuda.current_stream(dev)
    # copies on their own streams, pipelined across steps: step s+1's inputs
    # go host->device on two copy streams (two copy engines) as soon as step
    # s's commit has read its inputs, while step s's result comes back
    # device->host on a third (PCIe is full duplex); step s+1's commit waits
    # for its inputs and for that read-back (it rewrites the gradient)
    h2d = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    d2h = torch.cuda.Stream(dev)
    ev = {"commit": None, "d2h": None}

    kill = StepKill(-1 if args.no_fail else 1 + args.e2e_steps // 2,
                    min(VICTIM_BUCKET, args.buckets - 1))

    # BENCH_E2E_COPY=serial: every copy on the step's stream (A/B only)
    serial = os.environ.get("BENCH_E2E_COPY", "") == "serial"
    if serial:
        h2d, d2h = [stream, stream], stream

    def one(s):
        for cs in h2d:
            if ev["commit"] is not None and cs is not stream:
                cs.wait_event(ev["commit"])
        for i, m in enumerate(idx):
            with torch.cuda.stream(h2d[i % 2]):
                leaves[m].copy_(host[m], non_blocking=True)
        for cs in h2d:
            if cs is not stream:
                stream.wait_stream(cs)
        if ev["d2h"] is not None:
            stream.wait_event(ev["d2h"])
        kill.step = s
        eng.step(s, lambda m, rid: leaves[m], kill)
        ev["commit"] = torch.cuda.Event()
        ev["commit"].record(stream)
        d2h.wait_event(ev["commit"])
        with torch.cuda.stream(d2h):
            out_host.copy_(eng.grads[mine[0]], non_blocking=True)
        ev["d2h"] = torch.cuda.Event()
        ev["d2h"].record(d2h)

    one(0)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    a = torch.cuda.Event(enable_timing=True)
    z = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    ev["commit"] = a  # the first copies start inside the timed region
    for s in range(args.e2e_steps):
        one(s + 1)
    stream.wait_event(ev["d2h"])
    z.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(z) / args.e2e_steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    bi = M * numel * 4          # every microbatch gradient, summed over ranks
    bo = world * numel * 4      # one committed gradient per rank
    return {"value": M * TOKENS_PER_MB / (ms / 1e3), "unit": "tokens/s",
            "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "ms_per_step": ms,
            "steps": args.e2e_steps, "pinned": pinned,
            "failure": None if args.no_fail else "replica 3 during_sync:%d at timed step %d"
            % (min(VICTIM_BUCKET, args.buckets - 1), args.e2e_steps // 2),
            "pcie_gbs_per_gpu": (bi + bo) / world / (ms / 1e3) / 1e9}


def main():
    args = parse()
    # exactly one JSON line on stdout: libraries (NCCL's version banner at
    # lazy communicator init) print to fd 1, so route fd 1 to stderr and keep
    # a private descriptor for the result line
    out_fd = os.dup(1)
    os.dup2(2, 1)
    global print
    builtin_print = print

    def print(*a, **k):  # noqa: A001 - the result line goes to the saved stdout
        if a and isinstance(a[0], str) and a[0].startswith("{"):
            os.write(out_fd, (a[0] + "\n").encode())
        else:
            builtin_print(*a, **k)
    try:
        if args.impl == "reference":
            run_reference_arm(args)
        else:
            run_ours(args)
    finally:
        sys.stdout.flush()


if __name__ == "__main__":
    main()
