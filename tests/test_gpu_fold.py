"""Parity of the librcv.so data plane against the CPU oracle (bitwise).

Fold order is part of the contract (comm.py:191-198, test_comm.py:235-243),
so every comparison here is on raw bytes: -0.0 vs +0.0 and the last ulp
matter.  Sizes: small cases against the numpy oracle; full BASELINE sizes
(GPT-2 124M gradient, 1 GiB buckets) through exact-arithmetic properties.
"""

import numpy as np
import pytest
import torch

from paper_2605_11215_b200 import _lib
from oracle import fold

from golden_util import unhex

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
NP_DT = {torch.float32: np.float32, torch.float64: np.float64}


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


def host(t):
    return t.detach().cpu().numpy()


def test_golden_fold_vectors(golden):
    for case in golden["fold_vectors"]:
        dt = np.dtype(case["dtype"])
        views = [dev(unhex(v).astype(dt)) for v in case["inputs"]]
        contrib = [case["latch"] or r not in ("major_spare", "minor_spare")
                   for r in case["roles"]]
        _lib.masked_allreduce(views, contrib)
        want = unhex(case["result"]).astype(dt).tobytes()
        for v in views:   # every member, spares included, holds the total
            assert host(v).tobytes() == want, case["name"]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 8, 16, 33, 64])
def test_masked_allreduce_random(dtype, n):
    rng = np.random.default_rng(n * 7 + (dtype == torch.float64))
    for numel in (0, 1, 3, 5, 17, 1023, 4099, 65536 + 13):
        off = int(rng.integers(0, 5))       # misaligned bucket views
        arrs = [rng.standard_normal(numel + off).astype(NP_DT[dtype]) for _ in range(n)]
        for a in arrs:                       # sprinkle signed zeros
            a[rng.integers(0, numel + off, size=min(3, numel + off))] = -0.0
        contrib = [bool(rng.random() < 0.7) for _ in range(n)]
        want = fold.masked_fold([a[off:] for a in arrs], contrib)
        bufs = [dev(a) for a in arrs]
        views = [b[off:] for b in bufs]
        _lib.masked_allreduce(views, contrib)
        for v in views:
            assert host(v).tobytes() == want.tobytes(), (n, numel, off)
        for b, a in zip(bufs, arrs):        # nothing outside the views moved
            assert host(b)[:off].tobytes() == a[:off].tobytes()


@pytest.mark.parametrize("variant", [_lib.VARIANT_TMA, _lib.VARIANT_DIRECT, _lib.VARIANT_SCALAR])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_fold_variants_agree(variant, dtype):
    rng = np.random.default_rng(3)
    for n in (1, 2, 5, 8, 32):
        numel = 3 * 128 * 8 * 4 + 77
        xs = [rng.standard_normal(numel).astype(NP_DT[dtype]) for _ in range(n)]
        ops = [0] + [1] * (n - 1)
        want = fold.run_program(xs, ops, divisor=3.0)
        out = torch.empty(numel, dtype=dtype, device=DEV)
        _lib.fold([dev(x) for x in xs], ops, [out], divisor=3.0, variant=variant)
        assert host(out).tobytes() == want.tobytes(), (variant, n)


def test_divide_is_true_division():
    # x / 3 differs from x * (1/3) in the last ulp for many x
    x = np.arange(1, 100001, dtype=np.float32) * np.float32(0.37)
    out = torch.empty_like(dev(x))
    _lib.fold([dev(x)], [0], [out], divisor=3.0)
    assert host(out).tobytes() == (x / np.float32(3.0)).tobytes()
    assert (x / np.float32(3.0)).tobytes() != (x * np.float32(1 / 3.0)).tobytes()


@pytest.mark.parametrize("gdt", [torch.float32, torch.bfloat16])
def test_accumulate_order_and_canon(gdt):
    rng = np.random.default_rng(11)
    numel = 10007
    grads = [torch.from_numpy(rng.standard_normal(numel).astype(np.float32)).to(gdt)
             for _ in range(6)]
    grads[0][:5] = -0.0
    acc = torch.empty(numel, dtype=torch.float32, device=DEV)
    _lib.accumulate(acc, grads[0].to(DEV), first=True)
    # the first round is `zeros + grad` (trainer.py:192, 212): -0.0 -> +0.0
    assert not np.signbit(host(acc)[:5]).any()
    assert host(acc).tobytes() == fold.local_accumulate([grads[0].float().numpy()],
                                                        np.float32).tobytes()
    for g in grads[1:]:
        _lib.accumulate(acc, g.to(DEV), first=False)
    want = fold.local_accumulate([g.float().numpy() for g in grads], np.float32)
    assert host(acc).tobytes() == want.tobytes()


def test_accumulate_f64():
    rng = np.random.default_rng(12)
    gs = [rng.standard_normal(999) for _ in range(4)]
    acc = torch.empty(999, dtype=torch.float64, device=DEV)
    for j, g in enumerate(gs):
        _lib.accumulate(acc, dev(g), first=(j == 0))
    assert host(acc).tobytes() == fold.local_accumulate(gs).tobytes()


def _random_cover(rng, n_leaves):
    height = max(0, (n_leaves - 1).bit_length())
    blocks, pos = [], 0
    while pos < n_leaves:
        lev = int(rng.integers(0, height + 1))
        while pos % (1 << lev) or pos + (1 << lev) > (1 << height):
            lev -= 1
        if rng.random() < 0.85:
            blocks.append((pos, lev))
        pos += 1 << lev
    return blocks or [(0, 0)]


@pytest.mark.parametrize("variant", [_lib.VARIANT_AUTO, _lib.VARIANT_TMA, _lib.VARIANT_DIRECT])
@pytest.mark.parametrize("seed", range(6))
def test_tree_commit_matches_oracle(seed, variant):
    rng = np.random.default_rng(seed)
    n_leaves = int(rng.integers(1, 65))
    blocks = _random_cover(rng, n_leaves)[:64]
    numel = int(rng.integers(1, 20000))
    vals = [rng.standard_normal(numel).astype(np.float32) for _ in blocks]
    want = fold.tree_from_blocks([(v, lo, lev) for v, (lo, lev) in zip(vals, blocks)],
                                 max(n_leaves, blocks[-1][0] + (1 << blocks[-1][1])))
    want = want / np.float32(float(n_leaves))
    outs = [torch.empty(numel, dtype=torch.float32, device=DEV) for _ in range(3)]
    _lib.tree_commit([(dev(v), lo, lev) for v, (lo, lev) in zip(vals, blocks)],
                     max(n_leaves, blocks[-1][0] + (1 << blocks[-1][1])), outs,
                     float(n_leaves), variant=variant)
    for o in outs:
        assert host(o).tobytes() == want.tobytes()


def test_tree_commit_independent_of_assignment():
    """The committed gradient is a function of the microbatch gradients only:
    8 replicas x 4 microbatches, failure-free vs replica 3 lost and its four
    indices recomputed by survivors 0, 1, 2, 4 (SURVEY §8(d) accounting)."""
    rng = np.random.default_rng(50)
    numel, M = 50021, 32
    leaves = [rng.standard_normal(numel).astype(np.float32) for _ in range(M)]
    L = [dev(x) for x in leaves]
    # failure-free: each replica pre-sums its aligned block of 4 (K-ACC tree)
    parts = []
    for r in range(8):
        p = torch.empty(numel, dtype=torch.float32, device=DEV)
        _lib.tree_commit([(L[4 * r + j], j, 0) for j in range(4)], 4, [p], 0.0)
        parts.append((p, 4 * r, 2))
    a = torch.empty(numel, dtype=torch.float32, device=DEV)
    _lib.tree_commit(parts, M, [a], float(M))
    # failure: block 12..15 arrives as four level-0 leaves from four survivors
    parts2 = [q for q in parts if q[1] != 12]
    parts2 += [(L[12 + j], 12 + j, 0) for j in range(4)]
    parts2.sort(key=lambda q: q[1])
    b = torch.empty_like(a)
    _lib.tree_commit(parts2, M, [b], float(M))
    assert host(a).tobytes() == host(b).tobytes()
    want = fold.canonical_tree(dict(enumerate(leaves)), M) / np.float32(M)
    assert host(a).tobytes() == want.tobytes()
    # the reference's own order differs only by rounding (rtol 1e-5 contract)
    ref = fold.grouped_reference_sum([leaves[4 * r:4 * r + 4] for r in range(8)],
                                     [True] * 8, np.float32) / np.float32(M)
    np.testing.assert_allclose(host(a), ref, rtol=1e-5, atol=1e-6)


def test_full_size_exact_property():
    """GPT-2 124M gradient (124,439,808 fp32) x 8 replicas: integer-valued
    inputs make every association exact, so the kernel must equal the exact
    sum; -0.0/+0.0 and the spare mask are checked on the same launch."""
    d = 124_439_808
    g = torch.Generator(device=DEV).manual_seed(0)
    views = [torch.randint(-64, 65, (d,), generator=g, device=DEV).float() for _ in range(8)]
    contrib = [True] * 7 + [False]
    want = torch.zeros(d, dtype=torch.float32, device=DEV)
    for v, c in zip(views, contrib):
        if c:
            want += v
    spare_before = views[7].clone()
    _lib.masked_allreduce(views, contrib)
    for v in views:
        assert torch.equal(v, want)
    assert not torch.equal(spare_before, want)
    del views, want, spare_before
    torch.cuda.empty_cache()


def test_compare_counts_bitwise():
    a = torch.zeros(1003, dtype=torch.float32, device=DEV)
    b = a.clone()
    b[7] = -0.0
    b[1002] = 1.0
    assert int(_lib.count_differences(a, b).item()) == 2


def test_sgd_commit_matches_numpy():
    rng = np.random.default_rng(4)
    for dt in (np.float64, np.float32):
        p = rng.standard_normal(3001).astype(dt)
        f = rng.standard_normal(3001).astype(dt)
        P = dev(p)
        _lib.sgd_commit(P, dev(f), 7.0, 0.05)
        assert host(P).tobytes() == fold.sgd(p, f, 7, 0.05).tobytes()


def test_unit_lanes_bit_exact():
    for seed, idx, salt, n in [(0, 0, 4, 64), (7, 123, 1, 1001), (2 ** 31 - 1, 10 ** 9, 3, 7)]:
        out = torch.empty(n, dtype=torch.float64, device=DEV)
        base = (seed * 0x9E3779B97F4A7C15 + idx * 0xBF58476D1CE4E5B9
                + salt * 0x94D049BB133111EB) & ((1 << 64) - 1)
        _lib.unit_lanes(out, base, 2.0, -1.0)
        assert host(out).tobytes() == (fold.unit_lanes(seed, idx, salt, n) * 2.0 - 1.0).tobytes()
        _lib.unit_lanes(out, base, floor7=True)
        want = np.floor(fold.unit_lanes(seed, idx, salt, n) * 7.0) - 3.0
        assert host(out).tobytes() == want.tobytes()


@pytest.mark.multigpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n_views", [2, 3, 8, 10])
def test_multidevice_allreduce(dtype, n_views):
    """The drop-in collective over views on several GPUs: <= 8 contributors
    run the fused one-launch kernel (entry barrier, owner slice, exit
    barrier), more take barrier + fold + barrier; bitwise vs the oracle's
    ascending masked fold, with empty owner slices (numel < 8 per device),
    ragged tails and the /B divisor."""
    n_dev = torch.cuda.device_count()
    _lib.enable_peer_access(list(range(n_dev)))
    rng = np.random.default_rng(9 + n_views)
    for numel in (1, 5, 1000, 1 << 20 | 3):
        for divisor in (0.0, 3.0):
            arrs = [rng.standard_normal(numel).astype(dtype) for _ in range(n_views)]
            contrib = [i != 1 for i in range(n_views)]  # 10 views: 9 contributors
            want = fold.masked_fold(arrs, contrib)
            if divisor:
                want = want / dtype(divisor)
            views = [torch.from_numpy(a).to("cuda:%d" % (i % n_dev)) for i, a in enumerate(arrs)]
            for _ in range(2):  # the second call re-reduces the first's output
                _lib.masked_allreduce(views, contrib, divisor)
                for v in views:
                    torch.cuda.synchronize(v.device)
                    assert host(v).tobytes() == want.tobytes(), (numel, divisor)
                arrs = [host(v) for v in views]
                want = fold.masked_fold(arrs, contrib)
                if divisor:
                    want = want / dtype(divisor)


@pytest.mark.parametrize("variant", [_lib.VARIANT_AUTO, _lib.VARIANT_TMA, _lib.VARIANT_DIRECT])
def test_bf16_leaves_wide_path(variant):
    """fp32 commit of bf16 microbatch gradients (HSDP shard leaves): 8-wide
    vectors, every load 16 bytes; bitwise vs the oracle on the widened data,
    including misaligned starts and ragged tails."""
    rng = np.random.default_rng(21)
    for n_leaves, numel, off in ((8, 4099, 0), (32, 50001, 3), (5, 777, 1), (16, 1 << 16, 8)):
        raw = [torch.from_numpy(rng.standard_normal(numel + off).astype(np.float32)).to(torch.bfloat16)
               for _ in range(n_leaves)]
        views = [r.to(DEV)[off:] for r in raw]
        widened = {m: r[off:].float().numpy() for m, r in enumerate(raw)}
        width = 1 << max(0, (n_leaves - 1).bit_length())
        want = fold.canonical_tree(widened, width) / np.float32(n_leaves)
        outs = [torch.empty(numel + off, dtype=torch.float32, device=DEV)[off:] for _ in range(2)]
        _lib.tree_commit([(v, m, 0) for m, v in enumerate(views)], width, outs,
                         float(n_leaves), variant=variant)
        for o in outs:
            assert host(o).tobytes() == want.tobytes(), (variant, n_leaves, numel, off)


def _random_program(rng, n):
    """A random valid stack program over n inputs (include/rcv.h): after
    each push merge 0..(depth-1) times, ending with one value; depth <= 8."""
    ops, depth = [], 0
    for i in range(n):
        depth += 1
        last = i == n - 1
        if last:
            m = depth - 1
        else:
            m = int(rng.integers(0, depth))
            if depth - m > 7:              # keep within ProgStack<8>
                m = depth - 7
        depth -= m
        op = m | (0x40 if rng.random() < 0.2 else 0)
        ops.append(op)
    return ops


@pytest.mark.parametrize("variant", [_lib.VARIANT_AUTO, _lib.VARIANT_TMA, _lib.VARIANT_DIRECT, _lib.VARIANT_SCALAR])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_random_stack_programs(variant, dtype):
    rng = np.random.default_rng(17 + (dtype == torch.float64))
    for trial in range(12):
        n = int(rng.integers(1, 40))
        numel = int(rng.integers(1, 9000))
        ops = _random_program(rng, n)
        xs = [rng.standard_normal(numel).astype(NP_DT[dtype]) for _ in range(n)]
        for x in xs:
            x[rng.integers(0, numel, size=min(2, numel))] = -0.0
        div = float(rng.choice([0.0, 3.0, 7.0]))
        want = fold.run_program(xs, ops, divisor=div)
        out = torch.empty(numel, dtype=dtype, device=DEV)
        _lib.fold([dev(x) for x in xs], ops, [out], divisor=div, variant=variant)
        assert host(out).tobytes() == want.tobytes(), (variant, trial, ops)


def test_fixed_programs_of_degraded_covers():
    """Every degraded combine cover of configs[1]'s group (shapes.inc, from
    tools/cover_shapes.py) runs a compile-time straight-line evaluator; its
    result is bitwise the oracle tree, on sizes with ragged heads and tails."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "cover_shapes.json")) as f:
        shapes = json.load(f)
    assert shapes
    rng = np.random.default_rng(11)
    for sh in shapes:
        blocks = [tuple(b) for b in sh["cover"]]
        ops, _ = _lib.tree_program(blocks, sh["n_leaves"])
        assert list(ops) == sh["ops"]
        for numel in (64 * 37, 64 * 37 + 5, 3):
            vals = [rng.standard_normal(numel).astype(np.float32) for _ in blocks]
            want = fold.tree_from_blocks([(v, lo, lev) for v, (lo, lev) in zip(vals, blocks)],
                                         sh["n_leaves"]) / np.float32(sh["n_leaves"])
            outs = [torch.empty(numel, dtype=torch.float32, device=DEV) for _ in range(2)]
            _lib.tree_commit([(dev(v), lo, lev) for v, (lo, lev) in zip(vals, blocks)],
                             sh["n_leaves"], outs, float(sh["n_leaves"]))
            for o in outs:
                assert host(o).tobytes() == want.tobytes(), (sh, numel)
