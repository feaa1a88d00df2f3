"""``metrics/v1`` rows for GPU runs and the accounting-parity compare
(SURVEY §8(f)4).

Rows carry the reference's schema (sim.py:323-348), so a GPU run and a
reference run of the same schedule diff mechanically: ``compare_rows``
checks every accounting field the reference pins (contributions, roles,
events, counters, bucket epochs, world size, layout) and ignores the clock
fields, which are wall-clock here and a simulated cost model there
(sim.py:203-219).  ``elapsed`` is measured; ``throughput`` is the paper's
effective throughput, tokens / (elapsed * alive replicas * ranks per
replica) (sim.py:324-326).
"""

from __future__ import annotations

import json
from typing import Dict, Iterable, List, Optional, Tuple

# fields whose values must agree exactly with the reference's rows
ACCOUNTING = ("iteration", "w_cur", "g_cur", "epoch", "roles", "contributions",
              "contrib_total", "contrib_regular", "contrib_boundary", "boundary",
              "bucket_epochs", "rounds", "passes", "reduces", "rewinds", "events")
# measured here, simulated there: reported, never compared
CLOCK = ("elapsed", "clock", "throughput", "loss")


def metrics_row(out, elapsed: float, clock: float, tokens_per_microbatch: int = 4096,
                ranks_per_replica: int = 1, loss: Optional[float] = None) -> dict:
    """One row from an IterationOutcome (trainer.py) or CommitOutcome
    (commit.py); sim.py:323-348 field for field."""
    tokens = out.contrib_total * tokens_per_microbatch
    denom = elapsed * out.w_cur * ranks_per_replica
    it = getattr(out, "iteration", getattr(out, "step", None))
    return {
        "iteration": it,
        "loss": float(loss if loss is not None else getattr(out, "loss", 0.0)),
        "w_cur": out.w_cur,
        "g_cur": out.state.g_cur,
        "epoch": out.final_epoch,
        "roles": sorted([rid, role] for rid, role in out.roles.items()),
        "contributions": sorted([rid, c] for rid, c in out.contributions.items()),
        "contrib_total": out.contrib_total,
        "contrib_regular": out.contrib_regular,
        "contrib_boundary": out.contrib_boundary,
        "boundary": out.boundary_crossed,
        "bucket_epochs": list(out.bucket_epochs),
        "rounds": out.rounds,
        "passes": out.passes,
        "reduces": out.reduces,
        "rewinds": out.rewinds,
        "elapsed": elapsed,
        "clock": clock,
        "tokens": tokens,
        "throughput": tokens / denom if denom > 0 else 0.0,
        "events": out.events,
    }


def write_metrics(path: str, meta: dict, rows: Iterable[dict]) -> None:
    """Line-delimited, sorted keys, meta line first (sim.py:430-444)."""
    with open(path, "w") as f:
        f.write(json.dumps(dict(meta, schema="metrics/v1"), sort_keys=True) + "\n")
        for row in rows:
            f.write(json.dumps(row, sort_keys=True) + "\n")


def read_metrics(path: str) -> Tuple[dict, List[dict]]:
    """sim.py:447-455."""
    with open(path) as f:
        lines = [ln for ln in f.read().splitlines() if ln.strip()]
    if not lines:
        raise ValueError("empty metrics file %r" % path)
    meta = json.loads(lines[0])
    if meta.get("schema") != "metrics/v1":
        raise ValueError("not a metrics file: missing schema 'metrics/v1'")
    return meta, [json.loads(ln) for ln in lines[1:]]


def _norm(v):
    # JSON round trips turn tuples into lists; compare structurally
    return json.loads(json.dumps(v, sort_keys=True))


def compare_rows(ours: List[dict], ref: List[dict],
                 fields: Tuple[str, ...] = ACCOUNTING) -> List[str]:
    """Every accounting difference between two runs of the same
    (config, schedule), as human-readable strings; [] means bit-exact
    microbatch accounting."""
    diffs = []
    if len(ours) != len(ref):
        diffs.append("row count %d != %d" % (len(ours), len(ref)))
    for a, b in zip(ours, ref):
        for f in fields:
            if f not in a or f not in b:
                continue
            if _norm(a[f]) != _norm(b[f]):
                diffs.append("iteration %s: %s %r != %r" % (b.get("iteration"), f, a[f], b[f]))
    return diffs


class ScheduleInjector:
    """Replays schedule/v1 entries (step, replica, location) like the
    reference's Injector (sim.py:180-198): polled by phase, a during_sync
    entry fires on its bucket."""

    def __init__(self, entries: Iterable[Tuple[int, int, str]]):
        self.by_step: Dict[int, List[Tuple[int, str]]] = {}
        for step, replica, loc in entries:
            self.by_step.setdefault(int(step), []).append((int(replica), loc))
        self.step = -1

    def set_step(self, step: int) -> None:
        self.step = step

    def fire(self, phase, bucket=None):
        out = []
        for replica, loc in self.by_step.get(self.step, ()):
            kind, _, b = loc.partition(":")
            if kind == phase and (phase != "during_sync" or int(b) == bucket):
                out.append(replica)
        return out


def replay_experiment(w_init: int, g_init: int, iterations: int, k_buckets: int,
                      dim: int, model_kind: str, stream_seed: int, lr: float,
                      policy: str, entries, device="cuda:0",
                      tokens_per_microbatch: int = 4096, ranks_per_replica: int = 8):
    """sim.run_experiment's world (sim.py:379-413) on the device drop-in,
    returning metrics/v1 rows with wall-clock elapsed."""
    import time

    import torch

    from .comm import Communicator, EmptyMembership
    from .policy import assign_roles, initial_state
    from .trainer import AllReplicasDead, DataStream, ReplicaState, ToyModel, run_iteration

    members = list(range(w_init))
    state = initial_state(w_init, g_init)
    comm = Communicator(members, assign_roles(state, members))
    stream = DataStream(stream_seed, w_init, dim, model_kind, device=device)
    reps = {r: ReplicaState(r, ToyModel(model_kind, torch.zeros(dim, dtype=torch.float64,
                                                                 device=device)), k_buckets)
            for r in members}
    inj = ScheduleInjector(entries)
    rows, clock = [], 0.0
    for t in range(iterations):
        inj.set_step(t)
        t0 = time.perf_counter()
        try:
            out = run_iteration(t, reps, comm, state, stream, injector=inj,
                                policy_kind=policy, lr=lr)
        except (AllReplicasDead, EmptyMembership):
            break
        torch.cuda.synchronize()
        elapsed = time.perf_counter() - t0
        clock += elapsed
        state = out.state
        rows.append(metrics_row(out, elapsed, clock, tokens_per_microbatch,
                                ranks_per_replica, loss=out.loss))
    return rows
