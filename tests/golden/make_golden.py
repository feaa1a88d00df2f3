"""Generate golden fixtures from the reference implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``steadybatch`` from /root/reference/pkg/src, drives
``run_iteration`` through scripted and randomly generated failure schedules,
and writes tests/golden/scenarios.json: every IterationOutcome field (floats
as float.hex, arrays as lists of hex) per iteration, plus the schedule that
produced it.  The fixtures travel to the GPU box; the reference does not.
"""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _hexlist(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


class Scripted:
    """Fires each (phase, bucket, [rids]) entry once (the reference tests'
    ScriptedInjector contract, test_trainer.py:33-50)."""

    def __init__(self, plan):
        self.plan = [tuple(p) for p in plan]

    def fire(self, phase, bucket=None):
        hit = [e for e in self.plan
               if e[0] == phase and (phase != "during_sync" or e[1] == bucket)]
        self.plan = [e for e in self.plan if e not in hit]
        return [r for e in hit for r in e[2]]


def run_reference(sb, spec):
    """spec: dict(w, g, k, dim, kind, seed, spares, policy, lr, iters, plans)
    where plans maps iteration -> list of (phase, bucket, [rids])."""
    from steadybatch.comm import Communicator
    from steadybatch.policy import assign_roles, initial_state, policy_advancement
    from steadybatch.trainer import DataStream, ReplicaState, ToyModel, run_iteration

    w, g = spec["w"], spec["g"]
    members = list(range(w + spec["spares"]))
    state = initial_state(w, g)
    if spec["spares"]:
        state = policy_advancement(state, w_cur=len(members))
    comm = Communicator(members, assign_roles(state, members))
    stream = DataStream(spec["seed"], len(members), spec["dim"], spec["kind"])
    reps = {r: ReplicaState(r, ToyModel(spec["kind"], np.zeros(spec["dim"])), spec["k"])
            for r in members}
    rows = []
    for t in range(spec["iters"]):
        plan = spec["plans"].get(str(t)) or spec["plans"].get(t)
        inj = Scripted(plan) if plan else None
        try:
            out = run_iteration(t, reps, comm, state, stream, injector=inj,
                                policy_kind=spec["policy"], lr=spec["lr"])
        except Exception as exc:  # recorded: the oracle must raise alike
            rows.append({"error": type(exc).__name__})
            break
        state = out.state
        first = next(r for r in comm.members if reps[r].alive)
        rows.append({
            "iteration": out.iteration,
            "loss": float(out.loss).hex(),
            "update": _hexlist(out.committed_update),
            "contributions": sorted([int(r), int(c)] for r, c in out.contributions.items()),
            "contrib_total": out.contrib_total,
            "contrib_regular": out.contrib_regular,
            "contrib_boundary": out.contrib_boundary,
            "final_epoch": out.final_epoch,
            "w_cur": out.w_cur,
            "g_cur": out.state.g_cur,
            "roles": sorted([int(r), v] for r, v in out.roles.items()),
            "events": out.events,
            "admitted": sorted(int(i) for i in out.admitted_indices),
            "bucket_epochs": list(out.bucket_epochs),
            "rounds": out.rounds, "passes": out.passes,
            "reduces": out.reduces, "rewinds": out.rewinds,
            "boundary": out.boundary_crossed,
            "params": _hexlist(reps[first].model.params),
        })
    return rows


def scenario(name, w, g, k=2, dim=3, kind="constant", seed=7, spares=0,
             policy="static", lr=0.05, iters=1, plans=None):
    return dict(name=name, w=w, g=g, k=k, dim=dim, kind=kind, seed=seed,
                spares=spares, policy=policy, lr=lr, iters=iters,
                plans={str(t): p for t, p in (plans or {}).items()})


def scripted_scenarios():
    """The reference tests' own worlds (test_trainer.py:151-351), SURVEY
    §3.7's counter table, and the Appendix-E golden trace."""
    S = []
    S.append(scenario("failure_free_constant", 4, 2, seed=3, iters=3))
    S.append(scenario("failure_free_k3_linear", 4, 2, k=3, kind="linear", seed=7))
    S.append(scenario("during_sync_no_spare", 4, 2, seed=5,
                      plans={0: [("during_sync", 0, [1])]}))
    S.append(scenario("during_sync_with_spare", 4, 2, seed=9, spares=1,
                      plans={0: [("during_sync", 0, [1])]}))
    S.append(scenario("before_sync", 4, 2, seed=2,
                      plans={0: [("before_sync", None, [0])]}))
    S.append(scenario("after_sync", 4, 2, seed=6,
                      plans={0: [("after_sync", None, [3])]}))
    S.append(scenario("degenerate_trajectory", 4, 2, seed=8, iters=4,
                      plans={1: [("during_sync", 1, [2])]}))
    S.append(scenario("adaptive_short", 4, 2, seed=8, iters=3, policy="adaptive",
                      plans={1: [("before_sync", None, [2])]}))
    S.append(scenario("two_simultaneous", 6, 2, seed=4,
                      plans={0: [("during_sync", 0, [1, 4])]}))
    S.append(scenario("stacked_boundary", 5, 2, seed=13,
                      plans={0: [("during_sync", 0, [1]), ("after_sync", None, [2])]}))
    S.append(scenario("spare_discard", 4, 2, seed=23, spares=1,
                      plans={0: [("during_sync", 0, [2, 3])]}))
    S.append(scenario("linear_loose", 4, 2, kind="linear", seed=21, dim=2,
                      lr=0.1, iters=30, plans={5: [("during_sync", 0, [3])]}))
    S.append(scenario("minor_layout_w3", 3, 3, seed=11, spares=0, iters=2))
    for loc, plan in [("none", []), ("ds1_spare", [("during_sync", 1, [1])]),
                      ("ds1_nospare", [("during_sync", 1, [1])]),
                      ("after", [("after_sync", None, [1])]),
                      ("after_spare", [("after_sync", None, [1])]),
                      ("before", [("before_sync", None, [1])])]:
        sp = 1 if "spare" in loc and "nospare" not in loc else 0
        S.append(scenario("survey_3_7_" + loc, 4, 2, k=4, seed=1, spares=sp,
                          plans={0: plan} if plan else None))
    S.append(scenario("appendix_e", 32, 8, k=4, dim=4, seed=7, iters=4,
                      plans={1: [("during_sync", 1, [5])],
                             2: [("during_sync", 0, [29])]}))
    S.append(scenario("gpt2_accounting_w8g4k20", 8, 4, k=20, dim=40, seed=50,
                      iters=3, plans={1: [("during_sync", 7, [3])]}))
    S.append(scenario("blocking_reenter", 4, 2, k=3, seed=31, spares=2, iters=2,
                      plans={0: [("during_sync", 1, [0]), ("after_sync", None, [1])]}))
    S.append(scenario("minus_zero_linear_dim5", 5, 1, k=5, kind="linear", dim=5,
                      seed=99, iters=3, plans={1: [("during_sync", 2, [4])]}))
    # a spare promoted for replica 0 dies later in the same step and a second
    # spare is promoted for it (round-1 advisor finding, commit.py)
    S.append(scenario("promoted_spare_dies_same_step", 4, 2, k=4, seed=41, spares=2,
                      iters=2, plans={0: [("during_sync", 1, [0]), ("during_sync", 2, [4])]}))
    return S


def random_scenarios(n=48, seed=20261018):
    """Random schedules in the shape of the reference acceptance sweep
    (test_acceptance.py:47-77): deaths at all three locations."""
    rng = random.Random(seed)
    S = []
    for j in range(n):
        w = rng.randint(2, 12)
        g = rng.randint(1, 5)
        k = rng.randint(1, 4)
        spares = rng.choice((0, 0, 1, 2))
        kind = "constant" if rng.random() < 0.6 else "linear"
        iters = 4
        total = w + spares
        n_fail = rng.randint(1, min(total - 1, 4))
        victims = rng.sample(range(total), n_fail)
        plans = {}
        for v in victims:
            t = rng.randrange(iters)
            phase = rng.choice(("before_sync", "during_sync", "during_sync", "after_sync"))
            bucket = rng.randrange(k) if phase == "during_sync" else None
            plans.setdefault(t, []).append((phase, bucket, [v]))
        S.append(scenario("random_%02d" % j, w, g, k=k, dim=rng.randint(2, 6),
                          kind=kind, seed=rng.randrange(2 ** 31), spares=spares,
                          policy="static" if rng.random() < 0.85 else "adaptive",
                          lr=0.05, iters=iters, plans=plans))
    return S


def fold_vectors():
    """Known-answer vectors for the collective, from the reference tests
    (test_comm.py:23-47, 144-151, 235-243) plus -0.0 cases, evaluated by the
    reference's own Communicator."""
    from steadybatch.comm import Communicator, ReplicaRole

    cases = []

    def run(name, vals, roles=None, latch=False, dtype=np.float64):
        n = len(vals)
        comm = Communicator(range(n), roles=roles)
        comm.boundary_latch = latch
        views = {r: np.array(vals[r], dtype=dtype) for r in range(n)}
        comm.ulfm_allreduce(views)
        cases.append(dict(name=name, dtype=np.dtype(dtype).name,
                          inputs=[_hexlist(v) for v in vals],
                          roles=[(roles or {}).get(r, ReplicaRole.MAJOR).value for r in range(n)],
                          latch=latch, result=_hexlist(views[0])))

    M, MS = ReplicaRole.MAJOR, ReplicaRole.MAJOR_SPARE
    run("identical_inputs", [[1.0, 2.0]] * 4)
    run("spare_virtual_zero", [[2.0], [2.0], [2.0], [5.0]], {0: M, 1: M, 2: M, 3: MS})
    run("boundary_latch_admits_spare", [[1.0], [10.0]], {0: M, 1: MS}, latch=True)
    run("fold_order", [[1e16], [1.0], [-1e16]])
    run("fold_order_f32", [[1e8], [1.0], [-1e8]], dtype=np.float32)
    run("minus_zero_kept", [[-0.0, 1.0], [-0.0, -1.0]])
    run("minus_zero_single", [[-0.0]])
    run("all_spares_zero", [[3.0], [4.0]], {0: MS, 1: MS})
    run("spare_first", [[7.0], [-0.0], [-0.0]], {0: MS, 1: M, 2: M})
    return cases


def metrics_runs():
    """sim.run_experiment metrics/v1 rows (sim.py:323-348, 363-413) for
    schedules generated by the reference's own generator, plus the
    acceptance gate's golden trace and throughput configs
    (test_acceptance.py:339-375, 506-541)."""
    from steadybatch.sim import (CostModel, ExperimentConfig, FailureSchedule,
                                 GenerationSpec, InjectionPoint, ScheduleEntry,
                                 generate_schedule, run_experiment)
    runs = []

    def add(name, cfg, sched):
        res = run_experiment(cfg, sched)
        runs.append(dict(
            name=name,
            config=dict(w_init=cfg.w_init, g_init=cfg.g_init, iterations=cfg.iterations,
                        k_buckets=cfg.k_buckets, dim=cfg.dim, model_kind=cfg.model_kind,
                        stream_seed=cfg.stream_seed, lr=cfg.lr, policy=cfg.policy),
            entries=[[e.step, e.replica, e.location.serialize()] for e in sched.entries],
            rows=res.rows, aborted=res.aborted))

    add("appendix_e_golden_trace",
        ExperimentConfig(w_init=32, g_init=8, iterations=4, k_buckets=4, dim=4,
                         model_kind="constant", stream_seed=7, policy="static"),
        FailureSchedule(GenerationSpec(32, 8, 4, 0, 2, 1, 3),
                        [ScheduleEntry(1, 5, 0, InjectionPoint("during_sync", 1)),
                         ScheduleEntry(2, 29, 3, InjectionPoint("during_sync", 0))]))
    add("throughput_amortization",
        ExperimentConfig(w_init=8, g_init=4, iterations=18, k_buckets=4, dim=3,
                         model_kind="constant", stream_seed=3, policy="static",
                         cost=CostModel(0.01, 0.5, 0.05, 0.003)),
        FailureSchedule(GenerationSpec(8, 8, 4, 0, 2, 3, 10),
                        [ScheduleEntry(3, 5, 0, InjectionPoint("before_sync")),
                         ScheduleEntry(9, 2, 0, InjectionPoint("before_sync"))]))
    rng = random.Random(7)
    for j in range(10):
        w = rng.randint(3, 12)
        k = rng.randint(1, 4)
        spec = GenerationSpec(w_init=w, ranks_per_replica=8, k_buckets=k,
                              seed=rng.randrange(2 ** 31), count=rng.randint(1, min(w - 1, 4)),
                              step_lo=0, step_hi=6, weights=(1.0, 2.0, 1.0))
        cfg = ExperimentConfig(w_init=w, g_init=rng.randint(1, 6), iterations=6, k_buckets=k,
                               dim=rng.randint(2, 5),
                               model_kind=rng.choice(("constant", "linear")),
                               stream_seed=rng.randrange(2 ** 31),
                               policy=rng.choice(("static", "static", "adaptive")))
        add("generated_%d" % j, cfg, generate_schedule(spec))
    return runs


def main():
    sys.path.insert(0, REF)
    import steadybatch as sb
    doc = {"generated_by": "tests/golden/make_golden.py",
           "reference": REF, "numpy": np.__version__,
           "scenarios": [], "fold_vectors": fold_vectors(),
           "metrics_runs": metrics_runs()}
    for spec in scripted_scenarios() + random_scenarios():
        doc["scenarios"].append(dict(spec, rows=run_reference(sb, spec)))
    path = os.path.join(HERE, "scenarios.json")
    with open(path, "w") as f:
        json.dump(doc, f, separators=(",", ":"), sort_keys=True)
    print("wrote %s: %d scenarios, %d fold vectors"
          % (path, len(doc["scenarios"]), len(doc["fold_vectors"])))


if __name__ == "__main__":
    main()
