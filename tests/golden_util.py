"""Helpers shared by the oracle and GPU replay tests (no product imports)."""

import numpy as np


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs], dtype=np.float64)


def plans_of(spec):
    """{iteration: [(phase, bucket, [rids])]} from a golden scenario."""
    return {int(t): [(p, b, list(r)) for p, b, r in plan]
            for t, plan in spec["plans"].items()}


ACCOUNTING = ("contrib_total", "contrib_regular", "contrib_boundary",
              "final_epoch", "w_cur", "g_cur", "bucket_epochs", "rounds",
              "passes", "reduces", "rewinds", "boundary")


def events_norm(events):
    out = []
    for e in events:
        out.append({"failed": [int(x) for x in e["failed"]],
                    "contrib": int(e["contrib"]),
                    "at_boundary": bool(e["at_boundary"]),
                    "g_ext": None if e["g_ext"] is None else int(e["g_ext"]),
                    "n_bdry": None if e["n_bdry"] is None else int(e["n_bdry"]),
                    "promoted": [[int(r), str(v)] for r, v in e["promoted"]],
                    "epoch_after": int(e["epoch_after"])})
    return out


def assert_accounting(got: dict, want: dict, where: str):
    """Bit-exact microbatch accounting (the north star's quota contract)."""
    for key in ACCOUNTING:
        assert got[key] == want[key], "%s: %s %r != %r" % (where, key, got[key], want[key])
    assert got["contributions"] == want["contributions"], where
    assert got["roles"] == want["roles"], where
    assert got["admitted"] == want["admitted"], where
    assert events_norm(got["events"]) == events_norm(want["events"]), where
