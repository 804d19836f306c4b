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


def pytest_sessionfinish(session, exitstatus):
    """With a library built with -DIMASK_BOUNDS_CHECK=1 (tools/gpu_bounds_check.sh)
    the kernels count every window / pair-image read outside its range: report
    the count after the GPU tests and fail the session if it is not zero."""
    try:
        import ctypes

        import torch

        if not torch.cuda.is_available():
            return
        from paper_2412_10249_b200 import _lib

        if _lib._lib is None:
            return
        out = (ctypes.c_ulonglong * 4)()
        if _lib.lib().imask_debug_bounds(out, 0) != 1:
            return
        print(f"\n[bounds check] violations {out[0]} (first: site {out[1]}, index "
              f"{ctypes.c_longlong(out[2]).value}, limit {out[3]})")
        if out[0]:
            session.exitstatus = 1
    except Exception as exc:  # pragma: no cover
        print(f"\n[bounds check] not read: {exc}")


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
