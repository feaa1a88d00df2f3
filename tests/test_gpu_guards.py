"""Out-of-bounds checks of every data-plane kernel, without compute-sanitizer
(closed on this pool: runs under it left GPUs needing a reset).  SURVEY
§5.2's memcheck/initcheck intent, restated as bitwise tests:

* every input view sits inside a larger buffer whose guard bands (before and
  after the view) hold NaN: a read outside the view would turn the result
  NaN (or change its bits), which the oracle comparison catches;
* every output view sits inside a larger buffer whose guard bands hold a
  canary bit pattern: a write outside the view changes a canary;
* every output element is pre-filled with a different canary, so an element
  the kernel forgot to write (initcheck) fails the bitwise comparison too.

Offsets and sizes are ragged (odd element offsets, sizes around the 16- and
32-byte vector widths and the 64-element slice unit), so heads and tails of
the vector kernels and the scalar path are all exercised, for every variant
(TMA ring, DIRECT, pair, forest, fixed degraded-cover programs, K-ACC)."""

import json
import os

import numpy as np
import pytest
import torch

from paper_2605_11215_b200 import _lib
from oracle import fold

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
GUARD = 4096  # elements of guard band on each side
CANARY = 0x7FA11D0D  # a quiet-NaN bit pattern no fold produces


def _guarded_input(x: np.ndarray, off: int, dtype=torch.float32):
    """x placed at element `off` of a NaN-filled buffer; returns (view, base)."""
    base = torch.full((GUARD + off + x.size + GUARD,), float("nan"), dtype=dtype, device=DEV)
    v = base[GUARD + off:GUARD + off + x.size]
    v.copy_(torch.from_numpy(np.ascontiguousarray(x)).to(dtype))
    return v, base


def _guarded_output(n: int, off: int, dtype=torch.float32):
    """An output view inside a canary-filled buffer (the view too)."""
    base = torch.empty(GUARD + off + n + GUARD, dtype=dtype, device=DEV)
    if dtype == torch.float64:
        base.view(torch.int64).fill_(CANARY | (CANARY << 32))
    else:
        base.view(torch.int32).fill_(CANARY)
    return base[GUARD + off:GUARD + off + n], base, off


def _check_canaries(base: torch.Tensor, off: int, n: int):
    w = base.view(torch.int64 if base.dtype == torch.float64 else torch.int32).cpu().numpy()
    c = (CANARY | (CANARY << 32)) if base.dtype == torch.float64 else CANARY
    head, tail = w[:GUARD + off], w[GUARD + off + n:]
    assert (head == c).all(), "write before the output view at %s" % np.nonzero(head != c)[0][-5:]
    assert (tail == c).all(), "write past the output view at %s" % np.nonzero(tail != c)[0][:5]


SIZES = [1, 3, 4, 7, 8, 63, 64, 65, 127, 255, 256, 1021, 4096 + 3, 64 * 37 + 5]
OFFS = [0, 1, 3, 4, 8]


@pytest.mark.parametrize("variant", [_lib.VARIANT_AUTO, _lib.VARIANT_TMA, _lib.VARIANT_DIRECT,
                                     _lib.VARIANT_SCALAR])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_fold_stays_in_bounds(variant, dtype):
    rng = np.random.default_rng(3 + (dtype == torch.float64))
    npdt = np.float32 if dtype == torch.float32 else np.float64
    for numel in SIZES:
        for off in OFFS:
            n_in = int(rng.integers(1, 9))
            xs = [rng.standard_normal(numel).astype(npdt) for _ in range(n_in)]
            ops = [0] + [1] * (n_in - 1)  # ascending left fold
            want = fold.run_program(xs, ops, divisor=3.0)
            ins = [_guarded_input(x, off + i, dtype) for i, x in enumerate(xs)]
            outs = [_guarded_output(numel, off + j, dtype) for j in range(2)]
            _lib.fold([v for v, _ in ins], ops, [o for o, _, _ in outs], divisor=3.0,
                      variant=variant)
            for o, base, oo in outs:
                assert o.cpu().numpy().tobytes() == want.tobytes(), (variant, numel, off)
                _check_canaries(base, oo, numel)


@pytest.mark.parametrize("variant", [_lib.VARIANT_AUTO, _lib.VARIANT_TMA, _lib.VARIANT_DIRECT])
def test_tree_commit_stays_in_bounds(variant):
    """Perfect trees (DIRECT: ProgFull, two-vector pair kernel for <= 8
    nodes) and trees with absent leaves (ProgTree)."""
    rng = np.random.default_rng(9)
    for n_leaves, blocks in [(8, [(i, 0) for i in range(8)]), (4, [(0, 1), (2, 1)]),
                             (32, [(i, 0) for i in range(32)]),
                             (16, [(0, 2), (4, 0), (5, 0), (8, 3)]), (2, [(0, 0), (1, 0)])]:
        for numel in (5, 64, 65, 64 * 37 + 5, 8192 + 7):
            for off in (0, 1, 4):
                vals = [rng.standard_normal(numel).astype(np.float32) for _ in blocks]
                want = fold.tree_from_blocks([(v, lo, lev) for v, (lo, lev) in zip(vals, blocks)],
                                             n_leaves) / np.float32(n_leaves)
                ins = [_guarded_input(v, off) for v in vals]
                outs = [_guarded_output(numel, off + j) for j in range(3)]
                _lib.tree_commit([(t, lo, lev) for (t, _), (lo, lev) in zip(ins, blocks)],
                                 n_leaves, [o for o, _, _ in outs], float(n_leaves),
                                 variant=variant)
                for o, base, oo in outs:
                    assert o.cpu().numpy().tobytes() == want.tobytes(), (blocks, numel, off)
                    _check_canaries(base, oo, numel)


def test_fixed_programs_stay_in_bounds():
    with open(os.path.join(os.path.dirname(__file__), "golden", "cover_shapes.json")) as f:
        shapes = json.load(f)
    rng = np.random.default_rng(13)
    for sh in shapes[::3]:
        blocks = [tuple(b) for b in sh["cover"]]
        for numel, off in ((64 * 11, 0), (64 * 11 + 3, 1), (7, 4)):
            vals = [rng.standard_normal(numel).astype(np.float32) for _ in blocks]
            want = fold.tree_from_blocks([(v, lo, lev) for v, (lo, lev) in zip(vals, blocks)],
                                         sh["n_leaves"]) / np.float32(sh["n_leaves"])
            ins = [_guarded_input(v, off) for v in vals]
            outs = [_guarded_output(numel, off + j) for j in range(2)]
            _lib.tree_commit([(t, lo, lev) for (t, _), (lo, lev) in zip(ins, blocks)],
                             sh["n_leaves"], [o for o, _, _ in outs], float(sh["n_leaves"]))
            for o, base, oo in outs:
                assert o.cpu().numpy().tobytes() == want.tobytes(), (sh["cover"], numel, off)
                _check_canaries(base, oo, numel)


def test_bf16_inputs_stay_in_bounds():
    rng = np.random.default_rng(21)
    for numel in (1, 7, 8, 9, 64, 65, 1000, 64 * 37 + 5):
        for off in (0, 1, 2, 8):
            xs = [rng.standard_normal(numel).astype(np.float32) for _ in range(4)]
            bf = [torch.from_numpy(x).to(torch.bfloat16) for x in xs]
            want = fold.run_program([b.float().numpy() for b in bf], [0, 1, 1, 1])
            ins = []
            for i, b in enumerate(bf):
                base = torch.full((GUARD + off + i + numel + GUARD,), float("nan"),
                                  dtype=torch.bfloat16, device=DEV)
                v = base[GUARD + off + i:GUARD + off + i + numel]
                v.copy_(b.to(DEV))
                ins.append(v)
            o, obase, oo = _guarded_output(numel, off)
            _lib.fold(ins, [0, 1, 1, 1], [o])
            assert o.cpu().numpy().tobytes() == want.tobytes(), (numel, off)
            _check_canaries(obase, oo, numel)


def test_kacc_push_stays_in_bounds():
    """K-ACC reads backward's per-parameter segments in place and merges the
    carry chain into the deepest stack entry: no byte outside them moves."""
    rng = np.random.default_rng(5)
    sizes = [4, 12, 64, 260, 1024, 8]
    numel = sum(sizes)
    segs_np = [rng.standard_normal(s).astype(np.float32) for s in sizes]
    segs = [_guarded_input(x, 0)[0] for x in segs_np]
    flat = np.concatenate(segs_np)
    s0 = rng.standard_normal(numel).astype(np.float32)
    s1 = rng.standard_normal(numel).astype(np.float32)
    deep, dbase, _ = _guarded_output(numel, 4)
    deep.copy_(torch.from_numpy(s0).to(DEV))
    top = _guarded_input(s1, 0)[0]
    _lib.kacc_push(segs, [deep, top], deep)
    want = s0 + (s1 + flat)
    assert deep.cpu().numpy().tobytes() == want.astype(np.float32).tobytes()
    _check_canaries(dbase, 4, numel)
    fresh, fbase, _ = _guarded_output(numel, 0)
    _lib.kacc_push(segs, [], fresh)
    assert fresh.cpu().numpy().tobytes() == flat.tobytes()
    _check_canaries(fbase, 0, numel)


def test_masked_allreduce_views_stay_in_bounds():
    """The drop-in collective writes the total into every member view in
    place: each view has its own guard bands; spares' views are written but
    not read."""
    rng = np.random.default_rng(8)
    for numel in (3, 64, 65, 1000, 64 * 37 + 5):
        for off in (0, 1, 5):
            xs = [rng.standard_normal(numel).astype(np.float32) for _ in range(5)]
            contrib = [True, True, False, True, True]
            want = fold.masked_fold(xs, contrib)
            bases, views = [], []
            for i, x in enumerate(xs):
                v, base, _ = _guarded_output(numel, off + i)
                v.copy_(torch.from_numpy(x).to(DEV))
                bases.append(base)
                views.append(v)
            _lib.masked_allreduce(views, contrib)
            for i, (v, base) in enumerate(zip(views, bases)):
                assert v.cpu().numpy().tobytes() == want.tobytes(), (numel, off, i)
                _check_canaries(base, off + i, numel)
