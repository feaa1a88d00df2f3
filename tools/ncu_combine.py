#!/usr/bin/env python
"""The multi-process commit's owner-slice combine, reproduced in ONE process
over N GPUs so ncu can profile it (no cross-process spin flags; ordering by
stream synchronisation): every live rank's cover-node partial of a 24.9 MB
configs[1] bucket sits on its GPU, and the combine of owner slice q runs on
GPU q, reading every node's slice (peers' over NVLink) and storing the
result into every GPU's primary (peers' over NVLink) — the same kernel,
program and access pattern as rcv_plan_bucket's combine.

    python tools/ncu_combine.py --cover perfect          # failure-free, N = #GPUs
    python tools/ncu_combine.py --cover 15               # tests/golden/cover_shapes.json[15]

Prints one JSON line: the concurrent (all owners at once, CUDA events, min
of reps) time per combine and the algorithmic NVLink bytes per direction;
under ncu (--metrics nvlrx__bytes_data_user.sum,nvltx__...) each launch's
counters give the measured bytes.
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_11215_b200 import _lib  # noqa: E402
from paper_2605_11215_b200.dist import owner_slice  # noqa: E402

BUCKET = 124_439_808 // 20 // 64 * 64  # configs[1]'s bucket (6,221,952 fp32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cover", default="perfect")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--numel", type=int, default=BUCKET)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    if a.cover == "perfect":
        n = a.n or torch.cuda.device_count()
        lev = (32 // n).bit_length() - 1
        cover = [(q << lev, lev) for q in range(n)]
        owner = list(range(n))
        n_leaves = 32
    else:
        with open(os.path.join(ROOT, "tests", "golden", "cover_shapes.json")) as f:
            sh = json.load(f)[int(a.cover)]
        n, cover, owner, n_leaves = sh["world"], [tuple(c) for c in sh["cover"]], \
            sh["owner_slot"], sh["n_leaves"]
    if torch.cuda.device_count() < n:
        raise SystemExit("needs %d GPUs" % n)
    devs = list(range(n))
    _lib.enable_peer_access(devs)
    numel = a.numel
    g = torch.Generator().manual_seed(5)
    parts = [torch.randn(numel, generator=g).to("cuda:%d" % owner[i]) for i in range(len(cover))]
    prim = [torch.empty(numel, device="cuda:%d" % d) for d in devs]
    plans = []
    for q in devs:
        lo, hi = owner_slice(numel, q, n)
        blocks = [(p.data_ptr() + lo * 4, c[0], c[1], _lib.F32) for p, c in zip(parts, cover)]
        tp = _lib.TreePlan(blocks, n_leaves, [t.data_ptr() + lo * 4 for t in prim], _lib.F32,
                           float(n_leaves))
        plans.append((q, tp, hi - lo))

    def run():
        evs = []
        for q, tp, cnt in plans:
            with torch.cuda.device(q):
                s = torch.cuda.current_stream(q)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                tp.run(0, 0, cnt, s.cuda_stream)
                e1.record(s)
                evs.append((e0, e1))
        for d in devs:
            torch.cuda.synchronize(d)
        return max(e0.elapsed_time(e1) for e0, e1 in evs)

    for _ in range(3):
        run()
    ms = min(run() for _ in range(a.reps))
    # per owner q: reads the slices of the nodes held elsewhere, stores its
    # slice into the n-1 other primaries; the busiest direction bounds it
    sl = numel * 4 / n
    rx = [(sum(1 for i in range(len(cover)) if owner[i] != q) + (n - 1)) * sl for q in devs]
    tx = [(sum(1 for i in range(len(cover)) if owner[i] == q) * (n - 1) + (n - 1)) * sl
          for q in devs]
    worst = max(max(rx), max(tx))
    print(json.dumps({"cover": a.cover, "n": n, "nodes": len(cover), "numel": numel,
                      "program": "ProgFull" if a.cover == "perfect" else "ProgFixed (shapes.inc)",
                      "ms_concurrent": ms, "nvlink_bytes_rx_per_gpu": rx,
                      "nvlink_bytes_tx_per_gpu": tx,
                      "busiest_direction_gbs": worst / ms / 1e6,
                      "frac_of_770": worst / ms / 1e6 / 770.0}))


if __name__ == "__main__":
    main()
