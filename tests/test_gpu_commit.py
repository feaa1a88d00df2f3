"""The canonical commit engine (commit.py) on CUDA.

Accounting contract: for every golden scenario the engine's per-replica
contributions, roles, events, counters and bucket epochs equal the
reference's exactly (the quota assignment is bit-exact).  Numeric contract:
the committed gradient is bitwise the canonical tree of the B microbatch
gradients / B — the same bits as the failure-free run — and within 1e-5 of
the reference's own fold order.
"""

import numpy as np
import pytest
import torch

from paper_2605_11215_b200.commit import GradientCommit, aligned_bounds, block_cover
from oracle import fold

from golden_util import events_norm, plans_of

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


class Scripted:
    def __init__(self, plan):
        self.plan = list(plan)

    def fire(self, phase, bucket=None):
        hit = [e for e in self.plan
               if e[0] == phase and (phase != "during_sync" or e[1] == bucket)]
        self.plan = [e for e in self.plan if e not in hit]
        return [r for e in hit for r in e[2]]


def _leaves(b, numel, seed):
    rng = np.random.default_rng(seed)
    host = [rng.standard_normal(numel).astype(np.float32) for _ in range(b)]
    return host, [torch.from_numpy(h).to(DEV) for h in host]


def test_engine_accounting_matches_reference(golden):
    checked = 0
    for spec in golden["scenarios"]:
        b = spec["w"] * spec["g"]
        if b > 64 or spec["k"] > 8:
            continue
        numel = 64 * spec["k"] + 37
        host, dev = _leaves(b, numel, spec["seed"] % 1000)
        eng = GradientCommit(numel, spec["w"], spec["g"], spec["k"],
                             spares=spec["spares"], policy_kind=spec["policy"])
        plans = plans_of(spec)
        want_grad = fold.canonical_tree(dict(enumerate(host)), b) / np.float32(b)
        for t, wr in enumerate(spec["rows"]):
            where = "%s step %d" % (spec["name"], t)
            if "error" in wr:
                with pytest.raises(Exception):
                    eng.step(t, lambda m, rid: dev[m], Scripted(plans.get(t, [])))
                break
            out = eng.step(t, lambda m, rid: dev[m], Scripted(plans.get(t, [])))
            assert sorted([r, c] for r, c in out.contributions.items()) == wr["contributions"], where
            assert sorted([r, v] for r, v in out.roles.items()) == wr["roles"], where
            assert events_norm(out.events) == events_norm(wr["events"]), where
            for key in ("contrib_total", "contrib_regular", "contrib_boundary",
                        "final_epoch", "w_cur", "rounds", "passes", "reduces",
                        "rewinds", "bucket_epochs"):
                assert getattr(out, key) == wr[key], (where, key)
            assert out.state.g_cur == wr["g_cur"], where
            assert out.boundary_crossed == wr["boundary"], where
            if spec["policy"] == "static":
                # every index committed exactly once -> the failure-free bits
                assert sorted(i for v in out.admitted.values() for i in v) == list(range(b))
                for r in eng.comm.members:
                    assert eng.grads[r].cpu().numpy().tobytes() == want_grad.tobytes(), where
            checked += 1
    assert checked > 40


def test_failure_run_equals_failure_free_bitwise():
    """configs[1] in miniature: 8 replicas x 4, replica 3 killed on bucket 7
    of 20 — committed gradients identical to the failure-free run, and within
    rtol 1e-5 of the reference's fold order."""
    numel = 20 * 64 * 7 + 5
    host, dev = _leaves(32, numel, 3)
    free = GradientCommit(numel, 8, 4, 20)
    free.step(0, lambda m, rid: dev[m])
    hurt = GradientCommit(numel, 8, 4, 20)
    out = hurt.step(0, lambda m, rid: dev[m], Scripted([("during_sync", 7, [3])]))
    assert out.events[0]["contrib"] == 28 and out.events[0]["g_ext"] == 1
    assert out.events[0]["n_bdry"] == 3 and out.rewinds == 8 and out.passes == 2
    assert out.contributions == {0: 5, 1: 5, 2: 5, 4: 5, 5: 4, 6: 4, 7: 4}
    a = free.grads[0].cpu().numpy()
    for r in hurt.comm.members:
        assert hurt.grads[r].cpu().numpy().tobytes() == a.tobytes()
    ref = fold.grouped_reference_sum([host[4 * r:4 * r + 4] for r in range(8)],
                                     [True] * 8, np.float32) / np.float32(32)
    np.testing.assert_allclose(a, ref, rtol=1e-5, atol=1e-6)
    # next step: the advanced 7-replica layout (G=5, one minor at 2)
    out2 = hurt.step(1, lambda m, rid: dev[m])
    assert out2.contributions == {0: 5, 1: 5, 2: 5, 4: 5, 5: 5, 6: 5, 7: 2}
    assert hurt.grads[0].cpu().numpy().tobytes() == a.tobytes()


def test_dead_replica_buffers_never_read():
    """Poison the dead replica's microbatch buffers after it dies: nothing
    changes, because its indices are recomputed by survivors (here: served
    from the survivors' own copies)."""
    numel = 4 * 64 * 3
    host, dev = _leaves(8, numel, 4)
    poisoned = [d.clone() for d in dev]

    class KillAndPoison(Scripted):
        def fire(self, phase, bucket=None):
            out = super().fire(phase, bucket)
            if 1 in out:
                for m in (2, 3):          # replica 1's canonical range
                    poisoned[m].fill_(float("nan"))
            return out

    eng = GradientCommit(numel, 4, 2, 3)
    eng.step(0, lambda m, rid: poisoned[m] if rid == 1 else dev[m],
             KillAndPoison([("during_sync", 1, [1])]))
    want = fold.canonical_tree(dict(enumerate(host)), 8) / np.float32(8)
    for r in eng.comm.members:
        assert eng.grads[r].cpu().numpy().tobytes() == want.tobytes()


def test_block_cover_and_bounds():
    assert aligned_bounds(1000, 3) == [(0, 320), (320, 640), (640, 1000)]
    owner = {m: ("a" if m < 8 else "b") for m in range(16)}
    assert block_cover(owner, 16) == [(0, 3), (8, 3)]
    owner = {m: "a" for m in range(32)}
    assert block_cover(owner, 32) == [(0, 5)]
    owner = {m: m // 3 for m in range(8)}
    assert block_cover(owner, 8) == [(0, 1), (2, 0), (3, 0), (4, 1), (6, 1)]


@pytest.mark.multigpu
def test_engine_multidevice_placement():
    n = torch.cuda.device_count()
    numel = 64 * 20 + 11
    host = [np.random.default_rng(m).standard_normal(numel).astype(np.float32) for m in range(32)]
    place = {r: torch.device("cuda", r % n) for r in range(8)}
    per_dev = {d: [torch.from_numpy(h).to(d) for h in host] for d in set(place.values())}
    eng = GradientCommit(numel, 8, 4, 20, placement=place)
    eng.step(0, lambda m, rid: per_dev[place[rid]][m], Scripted([("during_sync", 3, [5])]))
    want = fold.canonical_tree(dict(enumerate(host)), 32) / np.float32(32)
    for r in eng.comm.members:
        torch.cuda.synchronize(place[r])
        assert eng.grads[r].cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("bucket", [0, 3, 5])
def test_committed_buckets_survive_boundary(monkeypatch, bucket):
    """A during_sync death at `bucket` sends the step through a boundary and
    a second pass.  Buckets committed before the death keep their outputs
    (same microbatch index set, same leaf bits) instead of being relaunched;
    the committed gradient and the accounting equal the relaunching path's
    and the failure-free canonical tree bit for bit."""
    w, g, k = 4, 2, 6
    b = w * g
    numel = 64 * k * 3 + 40
    host, dev = _leaves(b, numel, 77 + bucket)
    want = fold.canonical_tree(dict(enumerate(host)), b) / np.float32(b)
    outs = {}
    for reuse in ("1", "0"):
        monkeypatch.setenv("RCV_REUSE", reuse)
        eng = GradientCommit(numel, w, g, k)
        out = eng.step(0, lambda m, rid: dev[m], Scripted([("during_sync", bucket, [2])]))
        torch.cuda.synchronize()
        for rid in eng.comm.members:
            assert eng.grads[rid].cpu().numpy().tobytes() == want.tobytes(), (reuse, rid)
        outs[reuse] = out
    a, z = outs["1"], outs["0"]
    for f in ("contributions", "contrib_total", "events", "bucket_epochs", "reduces",
              "rewinds", "passes", "roles"):
        assert getattr(a, f) == getattr(z, f), f
    # losing one of 4 replicas mid-commit crosses the boundary: the
    # relaunching path commits every bucket again in the second pass, reuse
    # relaunches only the failed bucket and those after it
    assert a.boundary_crossed and z.boundary_crossed
    assert z.launches - a.launches == bucket


def test_full_size_configs1_failure_step_vs_torch_tree():
    """configs[1] at full size: the GPT-2 124M gradient (d = 124,439,808
    fp32), 8 replicas x 4 microbatches, 20 buckets, replica 3 killed during
    the sync of bucket 7.  The survivors regenerate the dead replica's
    microbatch gradients (their own buffers, the same seeded values) and every
    survivor's committed gradient must equal, bitwise, the canonical tree
    evaluated independently with plain torch fp32 adds level by level and a
    true division by 32 (no librcv on the reference side) — at every element.
    The next step (the advanced 7-replica layout) commits the same bits."""
    d, w, g, k = 124_439_808, 8, 4, 20
    b = w * g

    def make(m):
        gen = torch.Generator(device=DEV).manual_seed(4321 + m)
        return torch.randn(d, generator=gen, device=DEV, dtype=torch.float32)

    leaves = [make(m) for m in range(b)]
    regen = {}

    def leaf(m, rid):
        if m // g == 3 and rid != 3:          # taken over from the dead replica
            if m not in regen:
                regen[m] = make(m)
            return regen[m]
        return leaves[m]

    eng = GradientCommit(d, w, g, k)
    out = eng.step(0, leaf, Scripted([("during_sync", 7, [3])]))
    assert out.contrib_total == b and out.events[0]["failed"] == [3]
    assert sorted(regen) == [12, 13, 14, 15]
    torch.cuda.synchronize()
    chunk = 1 << 24
    for step in (0, 1):
        if step == 1:
            eng.step(1, leaf)
            torch.cuda.synchronize()
        for lo in range(0, d, chunk):
            hi = min(d, lo + chunk)
            vals = [t[lo:hi] for t in leaves]
            while len(vals) > 1:
                vals = [vals[i] + vals[i + 1] for i in range(0, len(vals), 2)]
            want = (vals[0] / float(b)).view(torch.int32)
            for r in eng.comm.members:
                bad = int((eng.grads[r][lo:hi].view(torch.int32) != want).sum())
                assert bad == 0, (step, r, lo, bad)
    del leaves, regen
    torch.cuda.empty_cache()
