"""Multi-process commit (one process per GPU, NVLink P2P): the committed
gradient on every rank equals the CPU oracle's canonical tree bit for bit,
with and without replica and whole-rank deaths, and every step's pool-stamp
check is clean (``check_peers`` raises on a stale or overwritten partial).
A test needs one GPU per rank and is skipped on smaller boxes."""

import numpy as np
import pytest
import torch

from mp_util import failed, need_gpus, spawn

pytestmark = [pytest.mark.gpu]


class Kill:
    def __init__(self, plan):
        self.plan = list(plan)

    def fire(self, phase, bucket=None):
        hit = [e for e in self.plan if e[0] == phase and (phase != "during_sync" or e[1] == bucket)]
        self.plan = [e for e in self.plan if e not in hit]
        return [r for e in hit for r in e[2]]


def _bad_buckets(eng, want):
    bad = set()
    for r in eng.comm.members:
        if eng._holds(r):
            got = eng.grads[r].cpu().numpy()
            bad |= {j for j, (lo, hi) in enumerate(eng.bounds)
                    if got[lo:hi].tobytes() != want[lo:hi].tobytes()}
    return sorted(bad)


def _commit_worker(rank, world, combine_variant, multicast=False):
    from paper_2605_11215_b200.dist import DistributedGradientCommit
    from oracle import fold
    numel = 5 * 64 * 37 + 19
    host = [np.random.default_rng(100 + m).standard_normal(numel).astype(np.float32)
            for m in range(32)]
    dev = [torch.from_numpy(h).cuda() for h in host]
    want = fold.canonical_tree(dict(enumerate(host)), 32) / np.float32(32)
    eng = DistributedGradientCommit(numel, 8, 4, 5, combine_variant=combine_variant,
                                    barrier_timeout_s=60.0, multicast=multicast)
    assert eng.multicast == multicast
    results = []
    for t, plan in enumerate([[], [("during_sync", 2, [3])], [], [("before_sync", None, [6])]]):
        out = eng.step(t, lambda m, rid: dev[m], Kill(plan))
        torch.cuda.synchronize()
        results.append((_bad_buckets(eng, want), out.contrib_total,
                        sorted(out.contributions.items())))
    eng.check_peers()
    return results


@pytest.mark.parametrize("combine_variant,world,multicast",
                         [(0, 4, False), (2, 4, False), (0, 2, False), (0, 2, True), (0, 4, True),
                          (1, 4, True)])
def test_distributed_commit_bitwise(combine_variant, world, multicast):
    """multicast: the combine's all-gather stores through an NVLS multicast
    object (multimem.st) instead of one store per live peer."""
    need_gpus(world)
    res = spawn(_commit_worker, world, combine_variant, multicast)
    assert not failed(res), failed(res)
    for r in range(world):
        for bad, total, _ in res[r]:
            assert not bad and total == 32, (r, res[r])
    assert res[0] == res[world - 1]
    # after replica 3 died: advanced 7-replica layout, G = 5 and a minor at 2
    assert res[0][2][2] == [(0, 5), (1, 5), (2, 5), (4, 5), (5, 5), (6, 5), (7, 2)]


def _hsdp_worker(rank, world):
    from paper_2605_11215_b200.dist import HSDPCommit
    from oracle import fold
    shards, reps, g = 2, world // 2, 8
    b = reps * g
    numel = 2 * 4 * 64 * 21 + 64
    hsdp = HSDPCommit(numel, shards, reps, g, 4, barrier_timeout_s=60.0)
    lo, hi = hsdp.bounds[hsdp.shard]
    full = [np.random.default_rng(500 + m).standard_normal(numel).astype(np.float32)
            for m in range(b)]
    # bf16 microbatch gradients (the FSDP reduce-scatter output), fp32 commit
    bf = [torch.from_numpy(x).to(torch.bfloat16) for x in full]
    mine = [t[lo:hi].contiguous().cuda() for t in bf]
    widened = {m: t[lo:hi].float().numpy() for m, t in enumerate(bf)}
    want = fold.canonical_tree(widened, b) / np.float32(b)
    res = []
    for t, plan in enumerate([[], [("during_sync", 1, [reps - 1])], []]):
        out = hsdp.step(t, lambda m, rid: mine[m], Kill(plan))
        torch.cuda.synchronize()
        ok = (hsdp.replica not in hsdp.engine.comm.members or
              hsdp.grad.cpu().numpy().tobytes() == want.tobytes())
        res.append((ok, out.contrib_total, out.w_cur))
    hsdp.engine.check_peers()
    return res


def test_hsdp_commit_bf16_bitwise():
    world = 4  # 2 shards x 2 replicas
    need_gpus(world)
    res = spawn(_hsdp_worker, world)
    assert not failed(res), failed(res)
    for r in range(world):
        assert all(ok for ok, _, _ in res[r]), res[r]
        assert [tot for _, tot, _ in res[r]] == [16, 16, 16]
        assert [w for _, _, w in res[r]] == [2, 1, 1]


def _one_replica_worker(rank, world, g, k, plans, numel):
    """One replica per rank, so a replica death is a whole-rank death: the
    dead rank stops joining barriers after one last barrier over the old
    membership (its in-flight combine read the survivors' pools)."""
    from paper_2605_11215_b200.dist import DistributedGradientCommit
    from oracle import fold
    b = world * g
    host = [np.random.default_rng(700 + m).standard_normal(numel).astype(np.float32)
            for m in range(b)]
    dev = [torch.from_numpy(h).cuda() for h in host]
    want = fold.canonical_tree(dict(enumerate(host)), b) / np.float32(b)
    eng = DistributedGradientCommit(numel, world, g, k, barrier_timeout_s=60.0)
    res = []
    for t, plan in enumerate(plans):
        out = eng.step(t, lambda m, rid: dev[m], Kill(plan))
        torch.cuda.synchronize()
        res.append((_bad_buckets(eng, want), out.contrib_total, out.w_cur,
                    sorted(out.contributions.items())))
    eng.check_peers()
    return res


@pytest.mark.parametrize("world", [2, 4])
def test_whole_rank_death_one_replica_per_rank(world):
    need_gpus(world)
    plans = [[], [("during_sync", 3, [1])], [], []]
    res = spawn(_one_replica_worker, world, 4, 6, plans, 6 * 64 * 29 + 64)
    assert not failed(res), failed(res)
    for r in range(world):
        assert all(not bad for bad, _, _, _ in res[r]), (r, res[r])
        assert [tot for _, tot, _, _ in res[r]] == [4 * world] * 4
        assert [w for _, _, w, _ in res[r]] == [world] + [world - 1] * 3


def _configs1_worker(rank, world, plans, numel, multicast=False):
    """configs[1]'s replica group (W=8, G=4, K=20) spread over the ranks."""
    from paper_2605_11215_b200.dist import DistributedGradientCommit
    from oracle import fold
    w, g, k = 8, 4, 20
    host = [np.random.default_rng(500 + m).standard_normal(numel).astype(np.float32)
            for m in range(w * g)]
    dev = [torch.from_numpy(h).cuda() for h in host]
    want = fold.canonical_tree(dict(enumerate(host)), w * g) / np.float32(w * g)
    eng = DistributedGradientCommit(numel, w, g, k, barrier_timeout_s=60.0, multicast=multicast)
    res = []
    for t, plan in enumerate(plans):
        out = eng.step(t, lambda m, rid: dev[m], Kill(plan))
        torch.cuda.synchronize()
        res.append((_bad_buckets(eng, want), out.contrib_total, out.w_cur,
                    sorted(out.contributions.items())))
    eng.check_peers()
    return res


@pytest.mark.parametrize("reuse,multicast", [("1", False), ("0", False), ("1", True)])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_configs1_whole_rank_death(world, reuse, multicast, monkeypatch):
    """configs[1] (W=8, G=4, K=20) over `world` ranks, every replica of rank
    1 killed during_sync on bucket 7: a whole-rank death.  This shape (at
    world 8, one replica per rank) once gave wrong bits on the failure step
    (round 1): the dead rank's last combine still read a survivor's pool
    set after the survivors' barriers had dropped it.  Fixed by the
    membership-transition barrier (include/rcv.h); the pool stamps make any
    recurrence raise."""
    need_gpus(world)
    monkeypatch.setenv("RCV_REUSE", reuse)
    per = 8 // world
    dead = list(range(per, 2 * per))
    plans = [[], [("during_sync", 7, dead)], []]
    res = spawn(_configs1_worker, world, plans, 20 * 64 * 5 + 64, multicast)
    assert not failed(res), failed(res)
    bad = {r: [x[0] for x in res[r]] for r in range(world) if any(x[0] for x in res[r])}
    assert not bad, bad
    for r in range(world):
        assert [x[1] for x in res[r]] == [32] * 3
        assert [x[2] for x in res[r]] == [8, 8 - per, 8 - per]
    # the failure step's census then the advanced layout: every survivor
    # commits exactly 32, the dead rank's replicas contribute nothing
    for r in range(world):
        assert all(c == 0 for rid, c in res[r][1][3] if rid in dead) or \
            not any(rid in dead for rid, _ in res[r][1][3])
        assert not any(rid in dead for rid, _ in res[r][2][3])
