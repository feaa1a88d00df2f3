"""Pin the CPU oracle against fixtures generated from the reference itself
(tests/golden/make_golden.py).  Runs everywhere (no reference, no GPU)."""

import numpy as np
import pytest

from oracle import fold
from oracle.protocol import OracleAllDead, OracleInvariant, ScriptedKills, World

from golden_util import assert_accounting, plans_of, unhex


def oracle_rows(spec):
    world = World(spec["w"], spec["g"], k=spec["k"], dim=spec["dim"],
                  kind=spec["kind"], seed=spec["seed"], spares=spec["spares"],
                  policy=spec["policy"], lr=spec["lr"])
    plans = plans_of(spec)
    rows = []
    for t in range(spec["iters"]):
        try:
            out = world.iterate(t, ScriptedKills(plans.get(t, [])))
        except (OracleAllDead, OracleInvariant) as exc:
            rows.append({"error": type(exc).__name__})
            break
        rows.append(out)
    return rows


def as_row(out):
    return dict(out, contributions=sorted([r, c] for r, c in out["contributions"].items()),
                roles=sorted([r, v] for r, v in out["roles"].items()))


def test_golden_scenarios_bitwise(golden):
    assert len(golden["scenarios"]) >= 60
    for spec in golden["scenarios"]:
        got = oracle_rows(spec)
        assert len(got) == len(spec["rows"]), spec["name"]
        for g, w in zip(got, spec["rows"]):
            where = "%s it %s" % (spec["name"], w.get("iteration"))
            if "error" in w:
                assert "error" in g, where
                continue
            g = as_row(g)
            assert_accounting(g, w, where)
            # the oracle restates numpy's own arithmetic: bitwise everywhere
            assert np.array_equal(g["update"], unhex(w["update"])), where
            assert np.array_equal(g["params"], unhex(w["params"])), where
            assert float(g["loss"]).hex() == w["loss"], where


def test_fold_vectors(golden):
    for case in golden["fold_vectors"]:
        dt = np.dtype(case["dtype"])
        views = [unhex(v).astype(dt) for v in case["inputs"]]
        contrib = [case["latch"] or r not in ("major_spare", "minor_spare")
                   for r in case["roles"]]
        got = fold.masked_fold(views, contrib)
        want = unhex(case["result"]).astype(dt)
        assert got.tobytes() == want.tobytes(), case["name"]


def test_fold_order_known_answer():
    # (1e16 + 1) + (-1e16) == 0 in ascending order (test_comm.py:235-243)
    v = [np.array([1e16]), np.array([1.0]), np.array([-1e16])]
    assert fold.masked_fold(v, [True] * 3)[0] == 0.0
    # the order is the result: folding the -1e16 in before the 1.0 keeps it
    assert fold.masked_fold([v[0], v[2], v[1]], [True] * 3)[0] == 1.0


def test_canonical_tree_matches_blocks():
    rng = np.random.default_rng(5)
    leaves = {m: rng.standard_normal(7).astype(np.float32) for m in range(13)}
    full = fold.canonical_tree(leaves, 13)
    # pre-sum aligned blocks and combine: identical bits
    blocks = [(fold.canonical_tree({0: leaves[m], 1: leaves[m + 1],
                                    2: leaves[m + 2], 3: leaves[m + 3]}, 4), m, 2)
              for m in (0, 4, 8)]
    blocks.append((leaves[12], 12, 0))
    assert fold.tree_from_blocks(blocks, 13).tobytes() == full.tobytes()


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13, 32])
def test_program_interpreter_left_fold(n):
    rng = np.random.default_rng(n)
    xs = [rng.standard_normal(9) for _ in range(n)]
    ops = [0] + [1] * (n - 1)
    assert fold.run_program(xs, ops).tobytes() == fold.masked_fold(xs, [True] * n).tobytes()


def test_splitmix_lanes_pinned():
    # g0 of the constant stream is integer valued in [-3, 3] (trainer.py:152)
    g0 = fold.constant_g0(3, 64)
    assert np.array_equal(g0, np.round(g0)) and g0.min() >= -3 and g0.max() <= 3
