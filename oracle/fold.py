"""numpy restatement of the data plane (test infrastructure; see __init__)."""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np


def masked_fold(views: Sequence[np.ndarray], contrib: Sequence[bool]) -> np.ndarray:
    """Communicator.ulfm_allreduce's sum (comm.py:191-198): a left fold in
    ascending member order over contributors only, starting from a copy of
    the first contributor (so -0.0 survives), zeros when nobody contributes."""
    total: Optional[np.ndarray] = None
    for v, c in zip(views, contrib):
        if not c:
            continue
        total = np.array(v, copy=True) if total is None else total + v
    if total is None:
        total = np.zeros_like(views[0])
    return total


def local_accumulate(grads: Sequence[np.ndarray], dtype=np.float64) -> np.ndarray:
    """A replica's flat after its rounds: zeros, then `flat += grad` in round
    order (trainer.py:192, 212, 225)."""
    flat = np.zeros(grads[0].shape[0], dtype=dtype)
    for g in grads:
        flat += g
    return flat


def grouped_reference_sum(groups: Sequence[Sequence[np.ndarray]],
                          contrib: Sequence[bool], dtype=np.float64) -> np.ndarray:
    """The reference's committed sum for per-replica microbatch lists:
    per-replica local fold, then the masked ascending fold
    (trainer.py:212 then comm.py:191-198)."""
    flats = [local_accumulate(g, dtype) if len(g) else np.zeros(
        groups[0][0].shape[0] if groups and groups[0] else 0, dtype=dtype)
        for g in groups]
    return masked_fold(flats, contrib)


def canonical_tree(leaves: Dict[int, np.ndarray], n_leaves: int) -> Optional[np.ndarray]:
    """Canonical dyadic tree over next_pow2(n_leaves) microbatch indices,
    empty leaves skipped: node = left + right when both
    sides hold something, else the non-empty side."""
    height = 0
    while (1 << height) < n_leaves:
        height += 1

    def node(level: int, lo: int):
        if level == 0:
            return leaves.get(lo)
        half = 1 << (level - 1)
        a, b = node(level - 1, lo), node(level - 1, lo + half)
        if a is None:
            return b
        if b is None:
            return a
        return a + b

    return node(height, 0)


def tree_from_blocks(blocks: Sequence[Tuple[np.ndarray, int, int]],
                     n_leaves: int) -> Optional[np.ndarray]:
    """Same tree when some subtrees arrive pre-summed as aligned dyadic block
    partials (value, lo, level)."""
    height = 0
    while (1 << height) < n_leaves:
        height += 1
    by_key = {(lo, level): v for v, lo, level in blocks}
    spans = [(lo, lo + (1 << level)) for _, lo, level in blocks]

    def node(level: int, lo: int):
        if (lo, level) in by_key:
            return by_key[(lo, level)]
        hi = lo + (1 << level)
        if not any(a < hi and b > lo for a, b in spans) or level == 0:
            return None
        half = 1 << (level - 1)
        a, b = node(level - 1, lo), node(level - 1, lo + half)
        if a is None:
            return b
        if b is None:
            return a
        return a + b

    return node(height, 0)


def run_program(inputs: Sequence[np.ndarray], ops: Sequence[int],
                divisor: float = 0.0) -> np.ndarray:
    """Interpreter for rcv_fold's stack program (include/rcv.h)."""
    stack: List[np.ndarray] = []
    for x, op in zip(inputs, ops):
        if op & 0x40:
            x = np.zeros_like(x) + x
        stack.append(np.array(x, copy=True))
        for _ in range(op & 0x3F):
            b = stack.pop()
            a = stack.pop()
            stack.append(a + b)
    assert len(stack) == 1
    out = stack[0]
    if divisor:
        out = out / out.dtype.type(divisor)
    return out


def commit_update(flat: np.ndarray, b: int) -> np.ndarray:
    """update = flat / float(b) (trainer.py:446); numpy keeps flat's dtype."""
    return flat / float(b)


def sgd(params: np.ndarray, flat: np.ndarray, b: int, lr: float) -> np.ndarray:
    """params -= lr * (flat / float(b)) (trainer.py:450)."""
    out = params.copy()
    out -= lr * (flat / float(b))
    return out


# ---- splitmix example synthesis (trainer.py:64-87) ----

_M64 = (1 << 64) - 1


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def unit_lanes(seed: int, index: int, salt: int, n: int) -> np.ndarray:
    origin = (seed * 0x9E3779B97F4A7C15 + index * 0xBF58476D1CE4E5B9
              + salt * 0x94D049BB133111EB) & _M64
    with np.errstate(over="ignore"):
        z = _mix(np.uint64(origin) + np.arange(n, dtype=np.uint64)
                 * np.uint64(0x9E3779B97F4A7C15))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def constant_g0(seed: int, dim: int) -> np.ndarray:
    """The constant stream's integer-valued g0 (trainer.py:152-155)."""
    g0 = np.floor(unit_lanes(seed, 0, 4, dim) * 7.0) - 3.0
    if not g0.any():
        g0[0] = 1.0
    return g0


def linear_example(seed: int, i: int, dim: int, wstar: np.ndarray):
    """(x, y) of example i on the linear stream (trainer.py:157, 165-168)."""
    lanes = unit_lanes(seed, i, 1, dim + 1) * 2.0 - 1.0
    x = lanes[:dim]
    return x, float(wstar @ x + 0.1 * lanes[dim])


def linear_wstar(seed: int, dim: int) -> np.ndarray:
    return unit_lanes(seed, 0, 3, dim) * 2.0 - 1.0
