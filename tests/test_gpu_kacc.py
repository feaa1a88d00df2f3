"""K-ACC (rcv_kacc_push, kacc.py): every stack node is bitwise the oracle's
canonical subtree over the microbatches it covers, whatever the push order
and range, with gradients arriving as per-parameter segments (f32 or bf16);
a replica holds at most floor(log2 G) + 1 nodes; and the engine commits the
same bits from K-ACC nodes as from the microbatch gradients themselves."""

import numpy as np
import pytest
import torch

from oracle import fold
from paper_2605_11215_b200 import _lib
from paper_2605_11215_b200.commit import GradientCommit
from paper_2605_11215_b200.kacc import KAccumulator, Pending, SlotPool, stack_bound

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _segments(flat: torch.Tensor, sizes):
    """Split a flat gradient into separately allocated per-parameter tensors
    (as backward returns them)."""
    out, pos = [], 0
    for s in sizes:
        out.append(flat[pos:pos + s].clone())
        pos += s
    return out


@pytest.mark.parametrize("order", ["ascending", "range_5_13", "extension"])
def test_nodes_are_canonical_subtrees(order):
    numel = 4 * 1000
    sizes = [768, 4, 2000, 1228]
    assert sum(sizes) == numel
    rng = np.random.default_rng(3)
    host = {m: rng.standard_normal(numel).astype(np.float32) for m in range(32)}
    host[6][:17] = -0.0   # signed zeros of a lone leaf survive
    seq = {"ascending": list(range(16)), "range_5_13": list(range(5, 13)),
           "extension": [0, 1, 2, 3, 12, 13, 4, 5]}[order]
    pool = SlotPool(numel, DEV)
    acc = KAccumulator(pool)
    for m in seq:
        acc.push(m, _segments(torch.from_numpy(host[m]).to(DEV), sizes))
    torch.cuda.synchronize()
    covered = set()
    for node in acc.stack:
        idx = range(node.lo, node.lo + (1 << node.level))
        assert set(idx) <= set(seq)
        covered |= set(idx)
        want = fold.canonical_tree({m - node.lo: host[m] for m in idx}, 1 << node.level)
        assert node.tensor.cpu().numpy().tobytes() == want.tobytes(), (node.lo, node.level)
    assert covered == set(seq)
    if order != "extension":
        assert len(acc.stack) <= stack_bound(len(seq)) - 1


def test_bf16_segments_widen_exactly():
    numel = 4 * 257
    rng = np.random.default_rng(5)
    bf = [torch.from_numpy(rng.standard_normal(numel).astype(np.float32)).to(torch.bfloat16)
          for _ in range(4)]
    acc = KAccumulator(SlotPool(numel, DEV))
    for m, t in enumerate(bf):
        acc.push(m, _segments(t.to(DEV), [4 * 57, 4 * 200]))
    torch.cuda.synchronize()
    want = fold.canonical_tree({m: t.float().numpy() for m, t in enumerate(bf)}, 4)
    assert len(acc.stack) == 1
    assert acc.stack[0].tensor.cpu().numpy().tobytes() == want.tobytes()


def test_rejects_misaligned_segments():
    acc = KAccumulator(SlotPool(10, DEV))
    with pytest.raises(_lib.RcvError):
        acc.push(0, [torch.zeros(6, device=DEV), torch.zeros(4, device=DEV)])


def test_engine_commits_same_bits_from_kacc_nodes():
    """GradientCommit with K-ACC leaves (Pending -> KNode) vs raw microbatch
    gradients, through a replica death (extension pushes onto survivors'
    stacks): identical committed bits, equal to the oracle tree / B."""
    w, g, k = 4, 4, 3
    b = w * g
    numel = 3 * 64 * 11 + 64
    rng = np.random.default_rng(9)
    host = [rng.standard_normal(numel).astype(np.float32) for _ in range(b)]
    dev = [torch.from_numpy(h).to(DEV) for h in host]
    want = fold.canonical_tree(dict(enumerate(host)), b) / np.float32(b)

    class Kill:
        def __init__(self):
            self.done = False

        def fire(self, phase, bucket=None):
            if phase == "during_sync" and bucket == 1 and not self.done:
                self.done = True
                return [2]
            return []

    pool = SlotPool(numel, DEV)
    accs = {r: KAccumulator(pool) for r in range(w)}
    done = {}

    def leaf(m, rid):
        if (m, rid) not in done:
            accs[rid].push(m, [dev[m]])
            done[(m, rid)] = Pending(accs[rid], m)
        return done[(m, rid)]

    eng = GradientCommit(numel, w, g, k)
    out = eng.step(0, leaf, Kill())
    torch.cuda.synchronize()
    assert out.boundary_crossed and out.contrib_total == b
    for r in eng.comm.members:
        assert eng.grads[r].cpu().numpy().tobytes() == want.tobytes()
    # O(log G) memory: every live replica ends with at most log2(G)+1 nodes
    assert max(len(a.stack) for r, a in accs.items() if r in eng.comm.members) <= stack_bound(g)
