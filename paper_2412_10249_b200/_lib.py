"""ctypes binding of the in-tree C-ABI library ``libimask_b200.so``.

The library is the product: every device computation of this package goes
through it. There is no CPU or eager-PyTorch fallback -- a missing library
raises at first use.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional

from .errors import DimensionMismatch

LIB_NAME = "libimask_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

IMASK_OK = 0
IMASK_EINVAL = 1
IMASK_EDIM = 2
IMASK_ELEVEL = 3
IMASK_ECUDA = 4
IMASK_SQDIST_SCRATCH = 298

_c_float_p = ctypes.POINTER(ctypes.c_float)
_vp = ctypes.c_void_p


class ImaskState(ctypes.Structure):
    _fields_ = [
        ("x", _vp),
        ("y", _vp),
        ("b", _vp),
        ("phi_sum", _vp),
        ("psi_sum", _vp),
        ("phi_tab", _vp),
        ("psi_tab", _vp),
        ("bp", _vp),
        ("y_next", _vp),
        ("xbar", _vp),
    ]


class ImaskPdhgState(ctypes.Structure):
    _fields_ = [("x", _vp), ("xbar", _vp), ("y", _vp), ("b", _vp), ("bp", _vp)]


class ImaskPdhgParams(ctypes.Structure):
    _fields_ = [("sigma", ctypes.c_double), ("tau", ctypes.c_double),
                ("theta", ctypes.c_double), ("mu_g", ctypes.c_double)]


class ImaskStepParams(ctypes.Structure):
    _fields_ = [("sigma", ctypes.c_double), ("mu", ctypes.c_double), ("mu_g", ctypes.c_double),
                ("g_kind", ctypes.c_int), ("tv_iters", ctypes.c_int), ("tv_tol", ctypes.c_double),
                ("tv_mu", ctypes.c_double), ("tv_scratch", ctypes.c_void_p)]


# name -> (restype, argtypes)
SIGNATURES = {
    "imask_version": (ctypes.c_char_p, []),
    "imask_last_error": (ctypes.c_char_p, []),
    "imask_last_launch_count": (ctypes.c_int, []),
    "imask_prox_tv_scratch_bytes": (ctypes.c_int64, [ctypes.c_int]),
    "imask_prox_tv_nonneg": (
        ctypes.c_int,
        [ctypes.c_int, _vp, _vp, ctypes.c_double, ctypes.c_double, ctypes.c_int,
         ctypes.c_double, _vp, _vp],
    ),
    "imask_probe_ffma_peak": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    "imask_probe_smem_peak": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    "imask_sq_dist": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, _vp, _vp]),
    "imask_metric_row": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, _vp, _vp]),
    "imask_reload_switches": (ctypes.c_int, []),
    "imask_debug_bounds": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]),
    "imask_plan_create": (
        ctypes.c_int,
        [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
            ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_double, ctypes.c_int,
            ctypes.POINTER(_vp),
        ],
    ),
    "imask_plan_create_list": (
        ctypes.c_int,
        [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
            ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), ctypes.c_int,
            ctypes.POINTER(ctypes.c_double), ctypes.c_double, ctypes.c_int,
            ctypes.POINTER(ctypes.c_void_p),
        ],
    ),
    "imask_plan_destroy": (ctypes.c_int, [_vp]),
    "imask_plan_symmetric": (ctypes.c_int, [_vp]),
    "imask_plan_scratch_bytes": (ctypes.c_int64, [_vp]),
    "imask_project": (
        ctypes.c_int, [_vp, ctypes.c_int, _vp, ctypes.c_int64, _vp, ctypes.c_int64, _vp]
    ),
    "imask_backproject": (
        ctypes.c_int, [_vp, ctypes.c_int, _vp, ctypes.c_int64, _vp, ctypes.c_int64, _vp]
    ),
    "imask_restrict": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "imask_prolong": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, _vp, ctypes.c_float, _vp]),
    "imask_compensate": (
        ctypes.c_int,
        [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double), _vp, _vp, _vp],
    ),
    "imask_sketch_forward": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp]),
    "imask_sketch_adjoint": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp]),
    "imask_draw_levels": (
        ctypes.c_int,
        [
            ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
            ctypes.c_int, ctypes.POINTER(ctypes.c_int32),
        ],
    ),
    "imask_uniform_at": (ctypes.c_double, [ctypes.c_uint64, ctypes.c_int64]),
    "imask_sketch_step": (
        ctypes.c_int,
        [_vp, ctypes.POINTER(ImaskState), ctypes.c_int, ctypes.POINTER(ImaskStepParams), _vp],
    ),
    "imask_step_adjoint": (ctypes.c_int, [_vp, ctypes.POINTER(ImaskState), ctypes.c_int, _vp]),
    "imask_step_wait_staging": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
    "imask_step_forward": (
        ctypes.c_int,
        [_vp, ctypes.POINTER(ImaskState), ctypes.c_int, ctypes.POINTER(ImaskStepParams), _vp],
    ),
    "imask_step_image": (
        ctypes.c_int,
        [_vp, ctypes.POINTER(ImaskState), ctypes.c_int, ctypes.POINTER(ImaskStepParams), _vp],
    ),
    "imask_resum": (ctypes.c_int, [_vp, ctypes.POINTER(ImaskState), _vp]),
    "imask_step_graph_create": (
        ctypes.c_int,
        [_vp, ctypes.POINTER(ImaskState), ctypes.c_int, ctypes.POINTER(ImaskStepParams),
         ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int)],
    ),
    "imask_graph_launch": (ctypes.c_int, [_vp, _vp]),
    "imask_graph_destroy": (ctypes.c_int, [_vp]),
    "imask_seq_step": (
        ctypes.c_int,
        [_vp, ctypes.POINTER(ImaskState), ctypes.c_int, ctypes.POINTER(ImaskStepParams),
         ctypes.c_double, _vp],
    ),
    "imask_pdhg_step": (
        ctypes.c_int,
        [_vp, ctypes.POINTER(ImaskPdhgState), ctypes.POINTER(ImaskPdhgParams), _vp],
    ),
    "imask_step_graph_update": (
        ctypes.c_int,
        [_vp, _vp, ctypes.POINTER(ImaskState), ctypes.c_int, ctypes.POINTER(ImaskStepParams)],
    ),
}

_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    """Load the library (once); raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_NAME} not found at {LIB_PATH}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (or make -C "
                "paper_2412_10249_b200/csrc). There is no CPU fallback."
            )
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == IMASK_OK:
        return
    msg = lib().imask_last_error().decode()
    if rc == IMASK_EDIM:
        raise DimensionMismatch(msg)
    if rc in (IMASK_EINVAL, IMASK_ELEVEL):
        raise ValueError(msg)
    raise RuntimeError(f"imask CUDA failure: {msg}")


def last_launch_count() -> int:
    return int(lib().imask_last_launch_count())
