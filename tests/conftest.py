import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running check")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def g_rng():
    return golden("rng.npz")


@pytest.fixture(scope="session")
def g_proj_small():
    return golden("proj_small.npz")


@pytest.fixture(scope="session")
def g_proj_A():
    return golden("proj_A.npz")


@pytest.fixture(scope="session")
def g_proj_D():
    return golden("proj_D_sampled.npz")


@pytest.fixture(scope="session")
def g_sketch():
    return golden("sketch.npz")


@pytest.fixture(scope="session")
def g_solver_A():
    return golden("solver_A.npz")


@pytest.fixture(scope="session")
def g_tv():
    return golden("tv.npz")


def rel_l2(a, b):
    a = np.asarray(a, dtype=float).ravel()
    b = np.asarray(b, dtype=float).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
