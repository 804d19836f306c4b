"""The C-ABI library loads on a CPU-only host, exports every symbol the header
declares, and its host-side functions (level RNG, argument validation) behave
like the reference. No device compute is issued here."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO
from paper_2412_10249_b200 import _lib
from paper_2412_10249_b200.errors import DimensionMismatch

HEADER = os.path.join(REPO, "include", "imask_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"IMASK_API\s+[\w\s\*]+?\b(imask_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("imask_plan_create", "imask_project", "imask_backproject", "imask_restrict",
                 "imask_prolong", "imask_compensate", "imask_sketch_step", "imask_draw_levels",
                 "imask_step_adjoint", "imask_step_forward", "imask_step_image", "imask_resum"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_version():
    assert b"sm_100a" in _lib.lib().imask_version()


def test_draw_levels_bit_exact(g_rng):
    seeds = [int(s) for s in g_rng["seeds"]]
    L = _lib.lib()
    for pname, p in (("u3", [1 / 3] * 3), ("u6", [1 / 6] * 6), ("p4", [0.3, 0.3, 0.2, 0.2]),
                     ("u7", [1 / 7] * 7)):
        cum = np.cumsum(p)
        for si, seed in enumerate(seeds):
            out = np.empty(5000, dtype=np.int32)
            rc = L.imask_draw_levels(
                seed & (2**64 - 1), 0, 5000, cum.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                cum.size, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            )
            assert rc == 0
            assert np.array_equal(out, g_rng[f"levels_{pname}_s{si}"].astype(np.int32))
    u = np.array([L.imask_uniform_at(12345, k) for k in range(256)])
    assert np.array_equal(u, g_rng["uniform_s12345"])


def test_draw_levels_offset_window(g_rng):
    from paper_2412_10249_b200.solvers import draw_levels

    cum = np.cumsum([1 / 6] * 6)
    full = g_rng["levels_u6_s2"].astype(np.int32)
    assert np.array_equal(draw_levels(12345, 1000, 500, cum), full[1000:1500])


def _create(side=16, n_angles=4, n_det=23, begin=0, end=None, r=1, probs=(1.0,)):
    end = n_angles if end is None else end
    dp = ctypes.POINTER(ctypes.c_double)
    c = np.cos(np.arange(begin, end) * np.pi / n_angles)
    s = np.sin(np.arange(begin, end) * np.pi / n_angles)
    p = np.asarray(probs, dtype=float)
    h = ctypes.c_void_p()
    rc = _lib.lib().imask_plan_create(side, n_angles, n_det, begin, end, c.ctypes.data_as(dp),
                                      s.ctypes.data_as(dp), r, p.ctypes.data_as(dp), 1.0, 0,
                                      ctypes.byref(h))
    return rc


@pytest.mark.parametrize(
    "kwargs,code,msg",
    [
        (dict(side=0), _lib.IMASK_EINVAL, "side must be positive"),
        (dict(begin=3, end=2), _lib.IMASK_EINVAL, "angle slab"),
        (dict(end=9), _lib.IMASK_EINVAL, "angle slab"),
        (dict(side=12, r=4, probs=(0.25,) * 4), _lib.IMASK_EINVAL, "not divisible by 2^(r-1) = 8"),
        (dict(r=2, probs=(0.5, 0.6)), _lib.IMASK_EINVAL, "expected 1"),
        (dict(r=2, probs=(1.2, -0.2)), _lib.IMASK_EINVAL, "positive"),
        (dict(r=8, probs=(0.125,) * 8, side=256), _lib.IMASK_EINVAL, "1..7"),
    ],
)
def test_plan_validation_before_any_device_call(kwargs, code, msg):
    rc = _create(**kwargs)
    assert rc == code
    assert msg in _lib.lib().imask_last_error().decode()


def test_status_mapping():
    L = _lib.lib()
    rc = L.imask_restrict(12, 5, None, None, None)
    assert rc == _lib.IMASK_EINVAL
    with pytest.raises(ValueError, match="not divisible by factor 5"):
        _lib.check(rc)
    rc = L.imask_compensate(12, 4, None, None, None, None)
    with pytest.raises(ValueError, match="2\\^\\(r-1\\)"):
        _lib.check(rc)
    assert issubclass(DimensionMismatch, ValueError)
