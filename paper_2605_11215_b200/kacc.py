"""K-ACC: the canonical dyadic accumulator of a replica.

The reference accumulates every microbatch gradient into one flat buffer,
``flat += grad`` (trainer.py:202-229).  Its rounding then depends on which
replica ran which microbatch.  The B200 design commits the canonical dyadic
tree over microbatch indices instead; K-ACC builds that tree's nodes while
the microbatches finish, so a replica never holds more than O(log G)
gradient-sized buffers:

* pushing microbatch m starts the leaf node (m, 0);
* while the stack's top is that node's left sibling (same level, adjacent,
  aligned), the two merge into their parent;
* the whole carry chain is one ``rcv_kacc_push`` launch that reads the new
  gradient straight from backward's per-parameter outputs and the c merged
  entries and writes the parent in place of the deepest one.

Every node on the stack is therefore a complete canonical subtree
(lo, level) of 2^level present microbatches, bitwise equal to the value the
fused commit computes for it, and the stack of a contiguous range is its
maximal aligned dyadic cover.  The commit (``GradientCommit``) evaluates the
top of the tree over these nodes instead of over every microbatch gradient.

Memory per replica: at most floor(log2(G)) + 1 nodes, plus one transient.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence

import torch

from . import _lib


@dataclass(eq=False)
class KNode:
    """A complete canonical-tree node: the subtree over microbatch indices
    [lo, lo + 2^level), all present, held in `tensor` (fp32, flat)."""
    lo: int
    level: int
    tensor: torch.Tensor

    def covers(self, m: int) -> bool:
        return self.lo <= m < self.lo + (1 << self.level)


class SlotPool:
    """Gradient-sized fp32 buffers shared by the accumulators of one device.
    Slots return to the pool once merged; reuse is stream-ordered (every
    accumulator launches on the device's current stream)."""

    def __init__(self, numel: int, device):
        self.numel, self.device = numel, torch.device(device)
        self.free: List[torch.Tensor] = []
        self.allocated = 0
        self.in_use = 0
        self.peak_in_use = 0

    def take(self) -> torch.Tensor:
        self.in_use += 1
        self.peak_in_use = max(self.peak_in_use, self.in_use)
        if self.free:
            return self.free.pop()
        self.allocated += 1
        return torch.empty(self.numel, dtype=torch.float32, device=self.device)

    def give(self, t: torch.Tensor) -> None:
        self.in_use -= 1
        self.free.append(t)

    @property
    def bytes_allocated(self) -> int:
        return self.allocated * self.numel * 4


class KAccumulator:
    """The binary-counter stack of one replica."""

    def __init__(self, pool: SlotPool):
        self.pool = pool
        self.stack: List[KNode] = []
        self.pushed: List[int] = []
        self.peak_depth = 0

    def reset(self) -> None:
        for node in self.stack:
            self.pool.give(node.tensor)
        self.stack = []
        self.pushed = []

    def push(self, m: int, grads: Sequence[torch.Tensor]) -> None:
        """Accumulate microbatch m's gradient (backward's per-parameter
        tensors, in flat order)."""
        if m in self.pushed:
            raise ValueError("microbatch %d pushed twice" % m)
        lo, level, c = m, 0, 0
        k = len(self.stack)
        while c < k and c < _lib.KACC_MAX_DEPTH:
            top = self.stack[k - 1 - c]
            if top.level == level and top.lo + (1 << level) == lo and top.lo % (2 << level) == 0:
                lo, level, c = top.lo, level + 1, c + 1
            else:
                break
        merged = self.stack[k - c:]
        out = merged[0].tensor if merged else self.pool.take()
        _lib.kacc_push(grads, [n.tensor for n in merged], out)
        for n in merged[1:]:
            self.pool.give(n.tensor)
        del self.stack[k - c:]
        self.stack.append(KNode(lo, level, out))
        self.pushed.append(m)
        self.peak_depth = max(self.peak_depth, len(self.stack))

    def node_of(self, m: int) -> KNode:
        for n in self.stack:
            if n.covers(m):
                return n
        raise KeyError("microbatch %d is not on this accumulator" % m)


class Pending:
    """What a leaf provider returns for a K-ACC microbatch: resolved by the
    commit engine to the stack node holding it once every admitted
    microbatch of the step's leaf set has been pushed."""

    __slots__ = ("acc", "m")

    def __init__(self, acc: KAccumulator, m: int):
        self.acc, self.m = acc, m

    def resolve(self) -> KNode:
        return self.acc.node_of(self.m)


def stack_bound(g: int) -> int:
    """Nodes a replica of G microbatches holds at most, plus the transient
    slot of a push (floor(log2 G) + 2)."""
    return max(1, g).bit_length() + 1


def memory_report(pools: Dict[object, SlotPool], accs: Dict[int, KAccumulator], g: int,
                  numel: int) -> dict:
    return {"slot_bytes": numel * 4,
            "slots_allocated": sum(p.allocated for p in pools.values()),
            "peak_slots_in_use": sum(p.peak_in_use for p in pools.values()),
            "peak_stack_depth_per_replica": max((a.peak_depth for a in accs.values()), default=0),
            "bound_per_replica": stack_bound(g),
            "fused_design_slots": g * len(accs)}
