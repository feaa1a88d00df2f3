"""The C ABI loads without a GPU and exports every symbol include/rcv.h
declares; host-only entry points (the tree program builder) are checked
against the oracle.  No device compute here."""

import ctypes
import os
import random
import re

import numpy as np
import pytest

from paper_2605_11215_b200 import _lib
from oracle import fold

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "rcv.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rcv_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_header():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTS)
    assert lib.rcv_version() >= 1


def test_device_count_without_gpu():
    n = ctypes.c_int(-1)
    assert _lib.load().rcv_device_count(ctypes.byref(n)) == 0
    assert n.value >= 0


def test_library_is_sm100a_only():
    out = os.popen("cuobjdump --list-elf %s 2>/dev/null" % _lib.LIB_PATH).read()
    assert "sm_100a" in out
    assert "sm_90" not in out


def _tree_eval_program(leaves, blocks, n_leaves):
    vals = [v for v, _, _ in blocks]
    ops, depth = _lib.tree_program([(lo, lev) for _, lo, lev in blocks], n_leaves)
    return fold.run_program(vals, ops), depth


@pytest.mark.parametrize("seed", range(20))
def test_tree_program_matches_oracle_tree(seed):
    rng = random.Random(seed)
    n_leaves = rng.randint(1, 64)
    height = max(0, (n_leaves - 1).bit_length())
    # random aligned block cover of a random subset of [0, 2^height)
    blocks, pos = [], 0
    gen = np.random.default_rng(seed)
    while pos < (1 << height) and len(blocks) < 64:
        lev = rng.randint(0, height)
        while pos % (1 << lev):
            lev -= 1
        if pos + (1 << lev) > (1 << height):
            lev = 0
        if rng.random() < 0.8:
            blocks.append((gen.standard_normal(5).astype(np.float32), pos, lev))
        pos += 1 << lev
    if not blocks:
        blocks = [(gen.standard_normal(5).astype(np.float32), 0, 0)]
    got, depth = _tree_eval_program(None, blocks, max(n_leaves, blocks[-1][1] + (1 << blocks[-1][2])))
    want = fold.tree_from_blocks(blocks, max(n_leaves, blocks[-1][1] + (1 << blocks[-1][2])))
    assert got.tobytes() == want.tobytes()
    assert depth <= height + 1


def test_tree_program_failure_free_layout():
    # 8 replicas x 4 microbatches: one level-2 block each -> balanced 3-level tree
    ops, depth = _lib.tree_program([(4 * r, 2) for r in range(8)], 32)
    assert ops == [0, 1, 0, 2, 0, 1, 0, 3] and depth == 4


def test_tree_program_rejects_bad_covers():
    with pytest.raises(_lib.RcvError):
        _lib.tree_program([(1, 1)], 8)          # misaligned
    with pytest.raises(_lib.RcvError):
        _lib.tree_program([(0, 2), (2, 0)], 8)  # overlap
    with pytest.raises(_lib.RcvError):
        _lib.tree_program([(8, 0)], 8)          # outside the tree


def test_cpu_tensors_fail_loudly():
    import torch
    a = torch.zeros(4, dtype=torch.float32)
    with pytest.raises(_lib.RcvError, match="no CPU fallback"):
        _lib.accumulate(a, a)
    with pytest.raises(_lib.RcvError):
        _lib.masked_allreduce([a, a], [True, True])


def test_pool_sets_switch(monkeypatch):
    """rcv_pool_sets: the partial-pool set count the allocator (dist.py) and
    the native runtime share; 4 by default, RCV_POOL_SETS clamped to 3..8."""
    monkeypatch.delenv("RCV_POOL_SETS", raising=False)
    assert _lib.pool_sets() == 4
    for v, want in (("3", 3), ("6", 6), ("8", 8), ("20", 8), ("1", 3)):
        monkeypatch.setenv("RCV_POOL_SETS", v)
        assert _lib.pool_sets() == want, v
