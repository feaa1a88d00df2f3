"""Host logic of the multi-process commit on CPU: a world-2 gloo group runs
the replicated control plane and the per-bucket plan on both ranks and
checks they agree (same decisions, same cover, disjoint owner slices)."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_11215_b200.commit import block_cover
import torch

from paper_2605_11215_b200.dist import (DistributedGradientCommit, _value_key, owner_slice,
                                        plan_bucket)
from paper_2605_11215_b200.kacc import KNode


def test_owner_slices_partition():
    for n in (0, 1, 63, 64, 65, 1000, 6221990):
        for nr in (1, 2, 3, 4, 7, 8):
            spans = [owner_slice(n, q, nr) for q in range(nr)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, z), (a2, _) in zip(spans, spans[1:]):
                assert z == a2 and a % 64 == 0


def test_plan_cache_key_covers_every_leaf_kind():
    # the native plan cache keys a leaf set by what the plan captures: a
    # microbatch gradient's address, a K-ACC node's subtree and address
    # (HSDP and the executor commit K-ACC nodes), nothing for a dead leaf
    t = torch.zeros(4)
    assert _value_key(None) == ()
    assert _value_key(t) == (t.data_ptr(), torch.float32)
    n = KNode(8, 2, t)
    assert _value_key(n) == (8, 2, t.data_ptr(), torch.float32)
    assert _value_key(KNode(12, 2, t)) != _value_key(n)


def test_plan_failure_layout():
    # 8 replicas x 4 microbatches on 2 ranks, replica 3 dead, its 4 indices
    # recomputed by survivors 0, 1, 2 (rank 0) and 4 (rank 1)
    rank_of = {r: r // 4 for r in range(8)}
    holder = {m: m // 4 for m in range(32)}
    for m, r in zip(range(12, 16), (0, 1, 2, 4)):
        holder[m] = r
    owner = {m: rank_of[r] for m, r in holder.items()}
    cover, slot_of = plan_bucket(owner, 32, [0, 1], pool_slots=8)
    assert cover == [(0, 3), (8, 2), (12, 1), (14, 0), (15, 0), (16, 4)]
    assert [slot_of[c][0] for c in cover] == [0, 0, 0, 0, 1, 1]
    with pytest.raises(RuntimeError):
        plan_bucket(owner, 32, [0], pool_slots=8)     # rank 1 is not live
    with pytest.raises(RuntimeError):
        plan_bucket(owner, 32, [0, 1], pool_slots=2)  # rank 0 needs 4 slots


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_11215_b200.comm import Communicator
    from paper_2605_11215_b200.policy import assign_roles, initial_state
    # replicated control plane: both ranks run the same failure schedule
    st = initial_state(8, 4)
    comm = Communicator(range(8), assign_roles(st, list(range(8))))
    for r in comm.members:
        comm.contrib_regular[r] = 4
    comm.mark_dead(3)
    rec = comm.ulfm_consensus().record
    rank_of = {r: r // (8 // world) for r in range(8)}
    owner = {m: rank_of[min(m // 4, 7)] for m in range(32) if m // 4 in comm.members}
    live = sorted({rank_of[r] for r in comm.members})
    cover, slot_of = plan_bucket(owner, 32, live, 8)
    mine = owner_slice(6221990, live.index(rank), len(live))
    got = [None] * world
    dist.all_gather_object(got, (rec.contrib, rec.at_boundary, cover,
                                 sorted(slot_of.items()), mine))
    dist.destroy_process_group()
    q.put((rank, got))


@pytest.mark.parametrize("world", [2, 4])
def test_replicated_plan_agrees(world):
    """Every rank of a gloo group runs the replicated control plane through
    replica 3's death and builds the bucket plan: identical decisions, cover
    and slots on every rank, owner slices that partition the bucket."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    views = res[0]
    for v in views[1:]:
        assert v[:4] == views[0][:4]      # same decision and plan on every rank
    assert views[0][0] == 28 and views[0][1] is True    # census of 7 survivors x 4
    spans = [v[4] for v in views]
    assert spans[0][0] == 0 and spans[-1][1] == 6221990
    for (a, z), (a2, _) in zip(spans, spans[1:]):
        assert z == a2 and a % 64 == 0


def test_dyadic_packing_minimises_cover():
    """_canonical_ranges packs each rank's count into aligned blocks: a
    partition of [0, sum) whose cover has sum-of-popcounts nodes (the
    minimum), e.g. 9 instead of 11 for the N=4 layout after replica 3 dies."""
    import random
    class Fake:
        _dyadic_ranges = DistributedGradientCommit._dyadic_ranges
        _canonical_ranges = DistributedGradientCommit._canonical_ranges

    def pack(f, counts):
        f.__dict__.pop("_ranges_memo", None)
        return f._canonical_ranges(counts)

    def cover_size(ranges, rank_of, b):
        owner = {i: rank_of[r] for r, ids in ranges.items() for i in ids}
        return len(block_cover(owner, b))

    f = Fake()
    f.rank_of = {r: r // 2 for r in range(8)}
    assert len(pack(f, [(0, 8), (1, 8)])[1]) == 8
    counts = [(0, 5), (1, 5), (2, 5), (4, 5), (5, 5), (6, 5), (7, 2)]
    got = pack(f, counts)
    contiguous, pos = {}, 0
    for r, q in counts:
        contiguous[r] = list(range(pos, pos + q))
        pos += q
    assert cover_size(contiguous, f.rank_of, 32) == 11
    assert cover_size(got, f.rank_of, 32) == 9
    rng = random.Random(3)
    for _ in range(300):
        world = rng.choice([2, 3, 4, 8])
        per = rng.choice([1, 2, 4])
        f.rank_of = {r: r // per for r in range(world * per)}
        counts = [(r, rng.randint(0, 9)) for r in range(world * per)]
        total = sum(q for _, q in counts)
        got = pack(f, counts)
        ids = sorted(i for v in got.values() for i in v)
        assert ids == list(range(total))
        assert all(len(got[r]) == q for r, q in counts)
        by_rank = {}
        for r, q in counts:
            by_rank[f.rank_of[r]] = by_rank.get(f.rank_of[r], 0) + q
        if total:
            # (absent leaves past `total` can merge a rank's last block
            # upward, so the popcount sum is an upper bound here)
            want = sum(bin(c).count("1") for c in by_rank.values())
            contiguous, pos = {}, 0
            for r, q in counts:
                contiguous[r] = list(range(pos, pos + q))
                pos += q
            got_n = cover_size(got, f.rank_of, total)
            assert got_n <= cover_size(contiguous, f.rank_of, total)
            if total <= 64:
                assert got_n <= want
