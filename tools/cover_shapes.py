#!/usr/bin/env python
"""Enumerate the combine trees the multi-process commit can meet, host-only.

Runs the engine's replicated control plane (GradientCommit.step with the
multi-process canonical ranges) on the CPU for configs[1]'s replica group
(W = 8, G = 4, K buckets) at N = 2, 4, 8 ranks under every schedule of up to
`--max-deaths` replica deaths at every injection point of a step and over
the following steps, and records each bucket commit's cover: the post-order
fold program (number of cover nodes, merges after each) of the tree the
owner-slice combine evaluates.  Writes paper_2605_11215_b200/csrc/shapes.inc:
one RCV_SHAPE(index, n, ops) per distinct program, so the combine of each of these
covers runs a straight-line, compile-time evaluator (ProgFixed) instead of
the heap-indexed ProgTree.

    python tools/cover_shapes.py            # regenerate shapes.inc
"""

import argparse
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_11215_b200 import _lib  # noqa: E402
from paper_2605_11215_b200.comm import Communicator  # noqa: E402
from paper_2605_11215_b200.commit import aligned_bounds  # noqa: E402
from paper_2605_11215_b200.dist import DistributedGradientCommit, plan_bucket  # noqa: E402
from paper_2605_11215_b200.policy import assign_roles, initial_state  # noqa: E402


class HostSim(DistributedGradientCommit):
    """The engine with its data plane replaced by a recorder."""

    def __init__(self, w, g, k, world):
        self.rank, self.world = 0, world
        per = w // world
        self.rank_of = {r: r // per for r in range(w)}
        self.state = initial_state(w, g)
        self.comm = Communicator(list(range(w)), assign_roles(self.state, list(range(w))))
        self.policy_kind = "static"
        self.numel = k * 64 * 8
        self.bounds = aligned_bounds(self.numel, k)
        self.alive = {r: True for r in range(w)}
        self.recovery_events = None
        self.real_kill = False
        self.pool_slots = 8
        self.shapes = set()
        self.examples = {}
        self.step_t, self.phase = -1, ""

    def _holds(self, rid):
        return True

    def _reduce_bucket(self, k, leaves):
        if not leaves:
            return 0
        ranks = sorted({self.rank_of[r] for r in self.comm.members})
        owner = {m: self.rank_of[rid] for m, (rid, _) in leaves.items()}
        cover, slot_of = plan_bucket(owner, self.state.b, ranks, self.pool_slots)
        if not _perfect(cover, self.state.b):
            ops, _ = _lib.tree_program(cover, self.state.b)
            key = (len(cover), tuple(ops))
            self.shapes.add(key)
            self.examples.setdefault(key, (self.state.b, list(cover),
                                           [ranks.index(slot_of[c][0]) for c in cover],
                                           self.world, self.step_t, self.phase))
        return 1

    def step(self, t, leaf, injector=None):
        self.step_t = t
        return super().step(t, leaf, injector)
        return 1

    def _end_of_step(self):
        pass


def _perfect(cover, b):
    """A perfect cover (equal nodes tiling the tree) runs ProgFull already."""
    lev = cover[0][1]
    return all(lv == lev and lo == i << lev for i, (lo, lv) in enumerate(cover)) and \
        len(cover) << lev == 1 << max(0, (b - 1).bit_length())


class Plan:
    def __init__(self, plan):
        self.plan = {t: list(v) for t, v in plan.items()}
        self.t = -1

    def fire(self, phase, bucket=None):
        cur = self.plan.get(self.t, [])
        hit = [e for e in cur if e[0] == phase and (phase != "during_sync" or e[1] == bucket)]
        self.plan[self.t] = [e for e in cur if e not in hit]
        return [r for e in hit for r in e[2]]


def schedules(w, k, max_deaths):
    points = [("before_sync", None), ("after_sync", None)] + [("during_sync", b)
                                                              for b in (0, k // 2, k - 1)]
    for n in range(1, max_deaths + 1):
        for victims in itertools.combinations(range(w), n):
            for pt in points:
                # all at once, and one per step
                yield {1: [(pt[0], pt[1], list(victims))]}
                if n > 1:
                    yield {1 + i: [(pt[0], pt[1], [v])] for i, v in enumerate(victims)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-deaths", type=int, default=1)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2605_11215_b200", "csrc",
                                                  "shapes.inc"))
    a = ap.parse_args()
    shapes = set()
    examples = {}
    w, g = 8, 4
    for world in (2, 4, 8):
        for plan in schedules(w, a.k, a.max_deaths):
            sim = HostSim(w, g, a.k, world)
            inj = Plan(plan)
            try:
                for t in range(4):
                    inj.t = t
                    sim.step(t, lambda m, rid: object(), inj)
            except Exception:
                pass  # a schedule that kills every replica of the group
            shapes |= sim.shapes
            for key, ex in sim.examples.items():
                examples.setdefault(key, ex)
    # programs the evaluator encodes: <= 16 inputs, <= 7 merges per input
    keep = sorted(s for s in shapes if s[0] <= 16 and all(o <= 7 for o in s[1]))
    with open(a.out, "w") as f:
        f.write("// generated by tools/cover_shapes.py: combine programs of configs[1]'s group\n"
                "// (W=8, G=4) at N=2/4/8 under up to %d replica deaths; RCV_SHAPE(index, n, ops)\n"
                "// with ops packed 3 bits per input (merges after pushing it)\n" % a.max_deaths)
        for i, (n, ops) in enumerate(keep):
            packed = sum(o << (3 * i) for i, o in enumerate(ops))
            f.write("RCV_SHAPE(%d, %d, 0x%xull)  // %s\n" % (i, n, packed, list(ops)))
    import json
    with open(os.path.join(ROOT, "tests", "golden", "cover_shapes.json"), "w") as f:
        json.dump([{"n_leaves": examples[s][0], "cover": examples[s][1], "ops": list(s[1]),
                    "owner_slot": examples[s][2], "world": examples[s][3]} for s in keep], f)
    print("%d distinct combine programs (%d kept) -> %s" % (len(shapes), len(keep), a.out))


if __name__ == "__main__":
    main()
