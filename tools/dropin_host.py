#!/usr/bin/env python
"""Host-side cost of the drop-in collective for small buckets: per call, the
time the caller's thread spends in Communicator.ulfm_allreduce, in
_lib.masked_allreduce alone, and in the bare C call (prepared ctypes
arguments), next to the device time of one call (CUDA events on every
device, max) and NCCL's all_reduce for the same tensors."""

import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11215_b200 import _lib  # noqa: E402
from paper_2605_11215_b200.comm import Communicator, ReplicaRole  # noqa: E402


def host_us(fn, devs, reps=200):
    for _ in range(10):
        fn()
    for d in devs:
        torch.cuda.synchronize(d)
    tot = 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        tot += time.perf_counter() - t0
        for d in devs:
            torch.cuda.synchronize(d)
    return tot / reps * 1e6


def dev_us(fn, devs, reps=50):
    best = 1e9
    for _ in range(reps):
        ev = {d: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for d in devs}
        for d in devs:
            ev[d][0].record(torch.cuda.current_stream(d))
        fn()
        for d in devs:
            ev[d][1].record(torch.cuda.current_stream(d))
        for d in devs:
            torch.cuda.synchronize(d)
        best = min(best, max(a.elapsed_time(z) for a, z in ev.values()) * 1e3)
    return best


def main():
    n_gpu = torch.cuda.device_count()
    for n in (2, 4):
        if n > n_gpu:
            continue
        for mb in (1, 4):
            numel = mb * (1 << 20) // 4
            devs = [torch.device("cuda", i) for i in range(n)]
            views = {r: torch.randn(numel, device=devs[r]) for r in range(n)}
            roles = {r: ReplicaRole.MAJOR for r in range(n)}
            comm = Communicator(list(range(n)), roles)
            _lib.enable_peer_access(list(range(n)))
            vl = [views[r] for r in range(n)]
            lib = _lib.load()
            ptrs = _lib._ptrs(vl)
            dev_arr = (ctypes.c_int * n)(*range(n))
            streams = (ctypes.c_void_p * n)(*[_lib.raw_stream(i) for i in range(n)])
            mask = (1 << n) - 1

            def bare():
                lib.rcv_masked_allreduce_multidev(ptrs, n, mask, _lib.F32, numel, 0.0, n, dev_arr, streams)
            import torch.cuda.nccl as nccl
            row = {"n": n, "mb": mb,
                   "host_us_ulfm_allreduce": host_us(lambda: comm.ulfm_allreduce(views), devs),
                   "host_us_masked_allreduce": host_us(lambda: _lib.masked_allreduce(vl, [True] * n), devs),
                   "host_us_bare_c_call": host_us(bare, devs),
                   "host_us_nccl": host_us(lambda: nccl.all_reduce(vl), devs),
                   "device_us_ulfm_allreduce": dev_us(lambda: comm.ulfm_allreduce(views), devs),
                   "device_us_bare_c_call": dev_us(bare, devs),
                   "device_us_nccl": dev_us(lambda: nccl.all_reduce(vl), devs)}
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
