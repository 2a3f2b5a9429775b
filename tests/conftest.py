"""Shared test fixtures.

Markers: ``gpu`` tests need a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on CPU.
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")
for p in (REPO, REPO / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (sm_100a)")


def has_cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def digest(*arrays):
    """SHA-256 of the arrays' bytes (tests/golden/make_golden.py's generator check)."""
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def reference_available():
    return (REFERENCE_SRC / "rbfdeform" / "core.py").exists()


def import_reference():
    """The reference package (only in the build container)."""
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    import rbfdeform

    return rbfdeform


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def cuda():
    if not has_cuda():
        pytest.fail("gpu-marked test selected but no CUDA device is visible")
    import paper_2004_04817_b200 as P

    return P
