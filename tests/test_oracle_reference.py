"""Oracle vs the live reference on fresh random schedules (build container
only: skipped where /root/reference is absent)."""

import random

import numpy as np
import pytest

from oracle import fold
from oracle.protocol import OracleAllDead, OracleInvariant, ScriptedKills, World, ext_rounds, layout


def _ref_world(sb, w, g, k, dim, kind, seed, spares, policy, lr):
    from steadybatch.comm import Communicator
    from steadybatch.policy import assign_roles, initial_state, policy_advancement
    from steadybatch.trainer import DataStream, ReplicaState, ToyModel
    members = list(range(w + spares))
    state = initial_state(w, g)
    if spares:
        state = policy_advancement(state, w_cur=len(members))
    comm = Communicator(members, assign_roles(state, members))
    stream = DataStream(seed, len(members), dim, kind)
    reps = {r: ReplicaState(r, ToyModel(kind, np.zeros(dim)), k) for r in members}
    return reps, comm, state, stream


@pytest.mark.parametrize("seed", range(4))
def test_oracle_matches_reference_random(reference, seed):
    from steadybatch.trainer import run_iteration
    rng = random.Random(1000 + seed)
    for _ in range(25):
        w, g, k = rng.randint(2, 10), rng.randint(1, 6), rng.randint(1, 5)
        spares = rng.choice((0, 1, 2))
        kind = rng.choice(("constant", "linear"))
        dim = rng.randint(1, 7)
        sd = rng.randrange(2 ** 31)
        policy = rng.choice(("static", "static", "adaptive"))
        reps, comm, state, stream = _ref_world(reference, w, g, k, dim, kind, sd,
                                               spares, policy, 0.05)
        world = World(w, g, k=k, dim=dim, kind=kind, seed=sd, spares=spares,
                      policy=policy)
        total = w + spares
        plans = {}
        for v in rng.sample(range(total), rng.randint(0, total - 1)):
            ph = rng.choice(("before_sync", "during_sync", "after_sync"))
            plans.setdefault(rng.randrange(4), []).append(
                (ph, rng.randrange(k) if ph == "during_sync" else None, [v]))
        for t in range(4):
            plan = plans.get(t, [])

            class Inj:
                def __init__(self, p):
                    self.k = ScriptedKills(list(p))

                def fire(self, phase, bucket=None):
                    return self.k.fire(phase, bucket)
            err_ref = err_or = None
            try:
                out = run_iteration(t, reps, comm, state, stream,
                                    injector=Inj(plan), policy_kind=policy)
                state = out.state
            except Exception as exc:
                err_ref = type(exc).__name__
            try:
                o = world.iterate(t, ScriptedKills(list(plan)))
            except (OracleAllDead, OracleInvariant) as exc:
                err_or = type(exc).__name__
            assert (err_ref is None) == (err_or is None), (err_ref, err_or)
            if err_ref:
                break
            assert o["contributions"] == out.contributions
            assert o["events"] == [dict(e, promoted=[list(p) for p in e["promoted"]])
                                   for e in out.events]
            assert o["bucket_epochs"] == out.bucket_epochs
            assert (o["rounds"], o["passes"], o["reduces"], o["rewinds"]) == \
                (out.rounds, out.passes, out.reduces, out.rewinds)
            assert o["update"].tobytes() == out.committed_update.tobytes()
            assert o["loss"] == out.loss


def test_policy_arithmetic_exhaustive(reference):
    """Oracle policy vs the reference's closed forms (cf. test_acceptance.py
    criterion 3), a reduced but complete grid."""
    from steadybatch.policy import extension_rounds, initial_state, policy_advancement
    for w in range(1, 33):
        for b in range(1, 257):
            st = initial_state(w, 1)
            st.b = b
            adv = policy_advancement(st, w_cur=w)
            lay = layout(w, b)
            assert (adv.g_cur, adv.n_maj, adv.r_cur, adv.n_min, adv.n_ms, adv.n_mi) == \
                (lay["g_cur"], lay["n_maj"], lay["r_cur"], lay["n_min"], lay["n_ms"], lay["n_mi"])
            for c in range(0, b + 1, max(1, b // 17)):
                assert int(extension_rounds(w, c, b)) == ext_rounds(w, c, b)


def test_splitmix_matches_reference(reference):
    from steadybatch.trainer import DataStream, _unit_lanes
    for seed in (0, 1, 7, 2 ** 31 - 1, 123456789):
        for idx in (0, 1, 99, 10 ** 9):
            assert _unit_lanes(seed, idx, 1, 33).tobytes() == fold.unit_lanes(seed, idx, 1, 33).tobytes()
        s = DataStream(seed, 4, 17, "constant")
        assert s.example(0)[0].tobytes() == fold.constant_g0(seed, 17).tobytes()
