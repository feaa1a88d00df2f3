"""Shared test plumbing.

Markers: ``gpu`` tests need a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on the CPU build container.
The reference (/root/reference) is imported only by tests marked with the
``reference`` fixture and is skipped where it is absent (the GPU box).
"""

import json
import os
import sys

# deterministic cuBLAS for the trajectory tests; must precede CUDA init
os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/pkg/src"
GOLDEN = os.path.join(ROOT, "tests", "golden", "scenarios.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
        n_gpu = torch.cuda.device_count() if have_gpu else 0
    except Exception:  # pragma: no cover
        have_gpu, n_gpu = False, 0
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    skip_multi = pytest.mark.skip(reason="needs >= 2 CUDA devices")
    for item in items:
        if "gpu" in item.keywords and not have_gpu:
            item.add_marker(skip_gpu)
        if "multigpu" in item.keywords and n_gpu < 2:
            item.add_marker(skip_multi)


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def reference():
    """The reference package ``steadybatch`` (build container only)."""
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not present (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import steadybatch
    return steadybatch
