"""Real-kill mode on >= 2 GPUs: rank 1's process SIGKILLs itself in the
middle of step 1's bucket cascade.  The survivors are not told: they find
out because their bounded barrier wait on rank 1 times out, mark its
replicas dead, and recover in-step (boundary extension, re-reduce over the
survivors).  Every committed gradient on every survivor — before, during
and after the failure — is bitwise the CPU oracle's canonical tree, i.e.
the failure-free result; no step is rolled back or replayed."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _worker(rank, world, port, q, per_bucket=False):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
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
        eng = DistributedGradientCommit(numel, w, g, 4, real_kill=True, barrier_timeout_s=1.0)
        inj = RealKill(1, "during_sync", 2) if rank == 1 else DeadPeerDetector(eng, shrink=True,
                                                                              per_bucket=per_bucket)
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
    # tearing the now-broken NCCL group down
    q.close()
    q.join_thread()
    os._exit(0)


@pytest.mark.parametrize("per_bucket", [False, True])
def test_real_process_death_recovered_in_step(per_bucket):
    world = min(torch.cuda.device_count(), 4)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, per_bucket)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world - 1):
        r, res, det = q.get(timeout=300)
        got[r] = (res, det)
    for p in procs:
        p.join(timeout=60)
    assert procs[1].exitcode == -9                 # the victim really died
    assert sorted(got) == [r for r in range(world) if r != 1]
    b = 4 * world
    for r, (res, det) in got.items():
        assert not isinstance(res, str), res
        assert all(ok for ok, _, _, _ in res), (r, res)
        assert [tot for _, tot, _, _ in res] == [b] * 4
        assert [wc for _, _, wc, _ in res] == [2 * world, 2 * world - 2, 2 * world - 2, 2 * world - 2]
        ev = res[1][3]
        assert len(ev) == 1 and ev[0]["failed"] == [2, 3] and ev[0]["at_boundary"]
        assert det and det[0]["ranks"] == [1]
        # per-bucket polling sees bucket 2's timed-out barrier before bucket 3
        want_at = ("during_sync", 3) if per_bucket else ("after_sync", None)
        assert (det[0]["phase"], det[0]["bucket"]) == want_at, det
