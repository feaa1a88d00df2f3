#!/usr/bin/env python
"""The reference's data path at the configs[1] size (GPT-2 124M fp32, 8
replicas x 4 microbatches, K=20), through the drop-in primitives on one GPU:
per-microbatch accumulation (trainer.py:212), per-bucket snapshot copies
(buckets.py:68) and the in-place ascending-fold collective
(comm.py:191-200), then update = flat / B (trainer.py:446).  Compared with
the fused canonical engine (commit.py) on the same inputs, failure-free.
Prints one JSON line."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_11215_b200 import _lib  # noqa: E402
from paper_2605_11215_b200.buckets import make_ledger, snapshot_and_tag  # noqa: E402
from paper_2605_11215_b200.comm import Communicator  # noqa: E402
from paper_2605_11215_b200.commit import GradientCommit  # noqa: E402

D, W, G, K, STEPS = 124_439_808, 8, 4, 20, 10


def main():
    dev = torch.device("cuda:0")
    gen = torch.Generator(device=dev).manual_seed(1234)
    leaves = [torch.randn(D, generator=gen, device=dev) for _ in range(W * G)]
    flats = [torch.empty(D, device=dev) for _ in range(W)]
    ledgers = [make_ledger(f, K) for f in flats]
    update = torch.empty(D, device=dev)

    def reference_path():
        for r in range(W):
            for j in range(G):
                _lib.accumulate(flats[r], leaves[r * G + j], first=(j == 0))
        comm = Communicator(range(W))
        for k in range(K):
            for led in ledgers:
                snapshot_and_tag(led, k, comm.epoch)
            comm.ulfm_allreduce({r: ledgers[r].buckets[k].data for r in range(W)})
        _lib.fold([flats[0]], [0], [update], divisor=float(W * G))

    eng = GradientCommit(D, W, G, K, placement={r: dev for r in range(W)})

    def engine_path():
        eng.step(0, lambda m, rid: leaves[m])

    out = {"config": "configs[1] size, failure-free step: GPT-2 124M fp32, 8 replicas x 4 "
                     "microbatches, K=20, one GPU"}
    for name, fn, nbytes in (("reference_order_dropin", reference_path, 114),
                             ("canonical_fused_engine", engine_path, 40)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(STEPS):
            fn()
        z.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(z) / STEPS
        out[name] = {"ms_per_step": ms, "algorithmic_hbm_bytes": nbytes * D * 4,
                     "hbm_gbs": nbytes * D * 4 / ms / 1e6}
    # the two orders commit the same gradient up to rounding (rtol 1e-5)
    ref_upd = update.clone()
    engine_path()
    torch.cuda.synchronize()
    diff = (eng.grads[0] - ref_upd).abs().max().item()
    out["max_abs_diff_reference_vs_canonical"] = diff
    out["speedup_fused_vs_reference_order"] = (out["reference_order_dropin"]["ms_per_step"]
                                               / out["canonical_fused_engine"]["ms_per_step"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
