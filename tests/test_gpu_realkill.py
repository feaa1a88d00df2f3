"""Real-kill mode: rank 1's process SIGKILLs itself in the middle of step
1's bucket cascade, with its kernels queued or running (no drain).  The
survivors are not told: the node liveness (native heartbeats in shared
memory) declares rank 1 dead within its deadline, every survivor's barrier
kernel stops waiting for it, and the survivors agree on the failed set at
the same protocol point (first rank to reach a poll decides it) and recover
in-step (boundary extension, re-reduce over the survivors).  Every committed
gradient on every survivor — before, during and after the failure — is
bitwise the CPU oracle's canonical tree, i.e. the failure-free result; no
step is rolled back or replayed.  One GPU per rank (two spinning ranks on
one GPU risk a context-switch timeout, B200_PROFILING.md), so it needs >= 2
devices."""

import os
import signal

import numpy as np
import pytest
import torch

from mp_util import free_port, init_rank

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _worker(rank, world, port, q):
    try:
        shared = init_rank(rank, world, port)
        from paper_2605_11215_b200.dist import (DeadPeerDetector, DistributedGradientCommit,
                                                RealKill)
        from oracle import fold
        w, g = 2 * world, 2
        b = w * g
        numel = 4 * 64 * 97 + 64
        host = [np.random.default_rng(900 + m).standard_normal(numel).astype(np.float32)
                for m in range(b)]
        dev = [torch.from_numpy(h).cuda() for h in host]
        want = fold.canonical_tree(dict(enumerate(host)), b) / np.float32(b)
        eng = DistributedGradientCommit(numel, w, g, 4, real_kill=True, barrier_timeout_s=30.0,
                                        liveness_deadline_s=20e-3)
        inj = RealKill(1, "during_sync", 2, liveness=eng.liveness) if rank == 1 else \
            DeadPeerDetector(eng, shrink=not shared)
        res = []
        for t in range(4):
            inj.step = t
            out = eng.step(t, lambda m, rid: dev[m], inj)
            torch.cuda.synchronize()
            ok = all(eng.grads[r].cpu().numpy().tobytes() == want.tobytes()
                     for r in eng.comm.members if eng._holds(r))
            res.append((ok, out.contrib_total, out.w_cur, out.events))
        q.put((rank, res, inj.detections))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc(), None))
    # flush the result (Queue.put is asynchronous), then leave without
    # tearing the now-broken process group down
    q.close()
    q.join_thread()
    os._exit(0)


def test_real_process_death_recovered_in_step():
    world = max(2, min(torch.cuda.device_count(), 4))
    port = free_port()
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world - 1):
        r, res, det = q.get(timeout=300)
        got[r] = (res, det)
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    # the victim really died (its traceback is in `got` if it raised instead)
    assert procs[1].exitcode == -signal.SIGKILL, got.get(1)
    assert sorted(got) == [r for r in range(world) if r != 1]
    b = 4 * world
    points = set()
    for r, (res, det) in got.items():
        assert not isinstance(res, str), res
        assert all(ok for ok, _, _, _ in res), (r, res)
        assert [tot for _, tot, _, _ in res] == [b] * 4
        assert [wc for _, _, wc, _ in res] == [2 * world, 2 * world - 2, 2 * world - 2, 2 * world - 2]
        ev = res[1][3]
        assert len(ev) == 1 and ev[0]["failed"] == [2, 3], ev
        assert det and det[0]["ranks"] == [1]
        assert det[0]["detect_ms"] <= 200, det      # deadline 20 ms (+ scheduling)
        points.add((det[0]["phase"], det[0]["bucket"], det[0]["poll"]))
    # agreement: every survivor acted on the death at the same protocol point
    assert len(points) == 1, points
