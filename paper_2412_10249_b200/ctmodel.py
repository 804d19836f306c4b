"""2-D parallel-beam projector on the B200 (drop-in for `mrtomo.ctmodel`).

Surface of the reference module for the hot path (pkg/src/mrtomo/ctmodel.py):
`Geometry` (ctmodel.py:38-70), `project` / `backproject` (ctmodel.py:170-185),
`projector_op` (ctmodel.py:188-191) and `coarse_projector`
(ctmodel.py:194-204). Instead of a cached scipy CSR matrix
(`_projector_pair`, ctmodel.py:157-167) each geometry gets a cached native
`Plan` holding float64-derived per-angle tables; the chords are evaluated on
the fly by the sm_100a kernels in `csrc/projector.cu`.

Phantoms, noise and the PGM I/O (ctmodel.py:207-333) are host-side data
tooling, out of scope for this path; the BASELINE's
synthetic inputs live in `synth.py`.
"""

from __future__ import annotations

import ctypes
import functools
import math
import os
import threading
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .linops import LinOp, default_device, to_device

AXIS_SNAP = 1e-14  # ctmodel.py:20


@dataclass(frozen=True)
class Geometry:
    """Parallel-beam scan geometry over a unit-pitch square grid (ctmodel.py:38-70)."""

    side: int
    n_angles: int = 100
    n_detectors: Optional[int] = None

    def __post_init__(self):
        if self.side < 1:
            raise ValueError("side must be positive")
        if self.n_detectors is None:
            object.__setattr__(
                self, "n_detectors", math.ceil(math.sqrt(2.0 * self.side * self.side))
            )

    @property
    def m(self) -> int:
        return self.n_angles * self.n_detectors

    @property
    def angles(self) -> np.ndarray:
        return np.arange(self.n_angles) * (np.pi / self.n_angles)

    @property
    def offsets(self) -> np.ndarray:
        n = self.n_detectors
        return np.arange(n, dtype=float) - (n - 1) / 2.0

    def cos_sin(self, begin: int = 0, end: Optional[int] = None, angles=None):
        """float64 cos/sin of angles [begin, end) (or of the index list ``angles``),
        snapped below 1e-14 (ctmodel.py:88-93).

        The snap is decided here, in float64, and passed to the device, so the
        axis-parallel tie rule never depends on float32 rounding.
        """
        if angles is not None:
            th = self.angles[np.asarray(angles, dtype=np.int64)]
        else:
            end = self.n_angles if end is None else end
            th = self.angles[begin:end]
        c = np.array([math.cos(t) for t in th])
        s = np.array([math.sin(t) for t in th])
        c[np.abs(c) < AXIS_SNAP] = 0.0
        s[np.abs(s) < AXIS_SNAP] = 0.0
        return c, s


def slab_bounds(n_angles: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous angle slab of one rank; uneven splits put the extra angles first."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n_angles, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


class _AngleTuple(tuple):
    """A tuple of Python ints that has been validated once (angle index lists
    are passed around per level and per call; re-converting 1440 entries each
    time was a third of make_problem's host time)."""


def _int_tuple(angles) -> "_AngleTuple":
    if type(angles) is _AngleTuple:
        return angles
    return _AngleTuple(int(a) for a in angles)


def shard_angles(n_angles: int, rank: int, world: int) -> tuple:
    """Mirror-closed angle shard of one rank (see _shard_angles; cached)."""
    return _shard_angles_cached(int(n_angles), int(rank), int(world),
                                os.environ.get("IMASK_SHARD_CYCLIC", "1"))


@functools.lru_cache(maxsize=256)
def _shard_angles_cached(n_angles: int, rank: int, world: int, _cyclic: str) -> tuple:
    return _AngleTuple(_shard_angles(n_angles, rank, world))


def _shard_angles(n_angles: int, rank: int, world: int) -> tuple:
    """Mirror-closed angle shard of one rank (global indices, local row order).

    Angle a and its mirror n_angles - a (theta -> pi - theta) always land on the
    same rank, so every rank runs the mirror-symmetric kernels. The base angles
    1..floor(n_angles/2) are split contiguously, balancing the row count (two
    rows per base, one for the self-mirrored pi/2 and for angle 0, which rank 0
    takes); angle counts divisible by 4 are split by quads (_shard_quads:
    block-cyclically when every rank gets at least four forward CTA groups).
    Row order: [0 on rank 0] + bases ascending + mirrors ascending,
    the layout imask_plan_create_list detects. world = 1 gives 0..n_angles-1.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if world == 1:
        return tuple(range(n_angles))
    if n_angles % 4 == 0 and n_angles >= 8:
        return _shard_quads(n_angles, rank, world)
    bases = list(range(1, n_angles // 2 + 1))
    weight = [1 if 2 * a == n_angles else 2 for a in bases]
    cum = np.concatenate([[1], 1 + np.cumsum(weight)])  # rows up to and including base i (+ angle 0)
    # rank k takes the bases whose cumulative row count falls in (k, k+1] * n_angles / world
    edges = [0] + [int(np.searchsorted(cum[1:], (k + 1) * n_angles / world - 0.5)) + 1
                   for k in range(world - 1)] + [len(bases)]
    edges = [min(max(e, 0), len(bases)) for e in edges]
    for k in range(1, len(edges)):
        edges[k] = max(edges[k], edges[k - 1])
    mine = bases[edges[rank]:edges[rank + 1]]
    mirrors = sorted(n_angles - a for a in mine if 2 * a != n_angles)
    return tuple(([0] if rank == 0 else []) + mine + mirrors)


_FWD_GROUP = 8  # entries per TMA forward CTA (projector.cu kFE)


def _shard_quads_cyclic(n_angles: int, rank: int, world: int):
    """Block-cyclic quad shards, or None where they do not apply.

    The whole set's forward entry list (capi.cu: the singles 0 and n/2, the
    quads of a = 1..n/4-1, the pair {n/4, 3n/4}) is cut into the groups of 8
    adjacent entries one forward CTA traces, and rank p takes the groups
    g = p (mod world): every rank gets the same mix of near-axis and oblique
    angles (a contiguous run gives rank 0 the near-axis ones, whose rays leave
    a third of the detector blocks empty), while a CTA's eight entries stay
    adjacent in angle, as its shared TMA windows need. Used when every rank
    gets >= 4 whole groups; the entries beyond the last whole cycle are cut
    into contiguous runs, so the row counts differ by a few rows only."""
    if os.environ.get("IMASK_SHARD_CYCLIC", "1") == "0":
        return None
    h, q = n_angles // 2, n_angles // 4
    n_entries = q + 2
    if n_entries // _FWD_GROUP < 4 * world:
        return None
    # whole cycles of groups go round-robin; the entries left over (fewer than
    # `world` groups) are cut into `world` contiguous runs, one short CTA each
    n_cyc = (n_entries // _FWD_GROUP // world) * world
    rest = n_entries - n_cyc * _FWD_GROUP
    lo = n_cyc * _FWD_GROUP + (rest * rank) // world
    hi = n_cyc * _FWD_GROUP + (rest * (rank + 1)) // world
    mine = [e for g in range(rank, n_cyc, world)
            for e in range(g * _FWD_GROUP, (g + 1) * _FWD_GROUP)] + list(range(lo, hi))
    low = set()
    for e in mine:
        if e == 0:
            continue  # angle 0: first row of its rank's list
        if e == 1:
            low.add(h)
        elif e == q + 1:
            low.add(q)
        else:
            low.update((e - 1, h - (e - 1)))
    low = sorted(low)
    mirrors = sorted(n_angles - a for a in low if a != h)
    return tuple(([0] if rank == 0 else []) + low + mirrors)


def _shard_quads(n_angles: int, rank: int, world: int) -> tuple:
    """shard_angles when n_angles % 4 == 0: shards closed under the mirror
    a -> n - a and the transpose a -> n/2 - a as well, so every rank's forward
    runs the four-ray (quad) TMA kernel. Units: the quads {a, n/2-a, n/2+a, n-a}
    (0 < a < n/4) split contiguously; rank 0 adds angles 0 and n/2, the last
    rank the pair {n/4, 3n/4}. Rows: [0] + the low angles (< n/2, and n/2)
    ascending + their mirrors ascending."""
    h, q = n_angles // 2, n_angles // 4
    quads = list(range(1, q))
    cyc = _shard_quads_cyclic(n_angles, rank, world)
    if cyc is not None:
        return cyc
    # rows before unit i: rank 0's two singles, four per quad; the pair adds 2 at the end
    cum = 2 + 4 * np.arange(1, len(quads) + 1)
    edges = [0] + [int(np.searchsorted(cum, (k + 1) * n_angles / world - 0.5)) + 1
                   for k in range(world - 1)] + [len(quads)]
    edges = [min(max(e, 0), len(quads)) for e in edges]
    for k in range(1, len(edges)):
        edges[k] = max(edges[k], edges[k - 1])
    mine = quads[edges[rank]:edges[rank + 1]]
    low = sorted(set(mine) | {h - a for a in mine}
                 | ({h} if rank == 0 else set()) | ({q} if rank == world - 1 else set()))
    mirrors = sorted(n_angles - a for a in low if a != h)
    return tuple(([0] if rank == 0 else []) + low + mirrors)


def quad_subset(n_angles: int, bases: Sequence[int]) -> tuple:
    """A sparse-view angle subset closed under the mirror a -> n - a and the
    transpose a -> n/2 - a (so the plan runs the four-ray forward and the
    mirror-symmetric adjoint): the quads {a, n/2-a, n/2+a, n-a} of the base
    angles 0 < a < n/4, plus 0, n/4, n/2 and 3n/4. Rows in the layout
    imask_plan_create_list recognises: [0] + low angles ascending + mirrors."""
    if n_angles % 4 != 0 or n_angles < 8:
        raise ValueError("quad subsets need n_angles divisible by 4 (and >= 8)")
    h, q = n_angles // 2, n_angles // 4
    bases = {int(a) for a in bases}
    if any(not 0 < a < q for a in bases):
        raise ValueError(f"base angles must lie in (0, {q})")
    low = sorted(bases | {h - a for a in bases} | {q, h})
    mirrors = sorted(n_angles - a for a in low if a != h)
    return tuple([0] + low + mirrors)


def _stream_ptr(device: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


@functools.lru_cache(maxsize=64)
def _full_range(begin: int, end: int) -> "_AngleTuple":
    return _AngleTuple(range(begin, end))


def _angle_list(geom: Geometry, angles=None, angle_begin: int = 0,
                angle_end: Optional[int] = None) -> tuple:
    if angles is not None:
        return _int_tuple(angles)
    angle_end = geom.n_angles if angle_end is None else angle_end
    return _full_range(angle_begin, angle_end)


class Plan:
    """Native plan of one geometry, angle set, sketch family and scale on one device.

    ``angles`` (global indices, local row order) selects this rank's sinogram
    rows; the default is all angles. ``angle_begin`` / ``angle_end`` select a
    contiguous slab instead.
    """

    def __init__(
        self,
        geom: Geometry,
        r: int = 1,
        probs: Sequence[float] = (1.0,),
        scale: float = 1.0,
        angle_begin: int = 0,
        angle_end: Optional[int] = None,
        device: Optional[torch.device] = None,
        angles=None,
    ):
        self.geom = geom
        self.device = device or default_device()
        self.angles = _angle_list(geom, angles, angle_begin, angle_end)
        self.n_loc = len(self.angles)
        self.m_loc = self.n_loc * geom.n_detectors
        self.r = int(r)
        self.probs = np.asarray(probs, dtype=float)
        self.scale = float(scale)
        self.factors = tuple(2 ** (self.r - i) for i in range(1, self.r + 1))
        c, s = geom.cos_sin(angles=self.angles)
        self._c = np.ascontiguousarray(c)
        self._s = np.ascontiguousarray(s)
        self._idx = np.ascontiguousarray(np.asarray(self.angles, dtype=np.int32))
        dp = ctypes.POINTER(ctypes.c_double)
        handle = ctypes.c_void_p()
        L = _lib.lib()
        with torch.cuda.device(self.device):
            _lib.check(
                L.imask_plan_create_list(
                    geom.side, geom.n_angles, geom.n_detectors, self.n_loc,
                    self._idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                    self._c.ctypes.data_as(dp), self._s.ctypes.data_as(dp), self.r,
                    self.probs.ctypes.data_as(dp), self.scale, self.device.index, ctypes.byref(handle),
                )
            )
        self.handle = handle
        self.graph_cache: dict = {}  # step graphs of solvers.Engine (destroyed with the plan)
        self.state_pool: list = []  # free solver-state buffers of run() (solvers.run)
        self.phi_offsets = []
        off = 0
        for f in self.factors:
            self.phi_offsets.append(off)
            # every row starts 16-byte aligned (imask_b200.h: imask_state.phi_tab)
            off = (off + (geom.side // f) ** 2 + 3) & ~3
        self.phi_tab_len = off

    def __del__(self):
        for g in getattr(self, "graph_cache", {}).values():
            try:
                _lib.lib().imask_graph_destroy(g[0])
            except Exception:
                pass
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.lib().imask_plan_destroy(h)
            except Exception:
                pass
            self.handle = None

    @property
    def symmetric(self) -> bool:
        """True when the mirror-symmetric kernels serve this plan's angle rows."""
        return _lib.lib().imask_plan_symmetric(self.handle) >= 1

    @property
    def quad_forward(self) -> bool:
        """True when the rows are also transpose-closed (four-ray TMA forward)."""
        return _lib.lib().imask_plan_symmetric(self.handle) == 2

    @property
    def stream(self) -> ctypes.c_void_p:
        return _stream_ptr(self.device)

    def project(self, u: torch.Tensor, factor: int, out: Optional[torch.Tensor] = None):
        """sino = R_f u on this slab (float32 device tensors)."""
        if out is None:
            out = torch.empty(self.m_loc, device=self.device, dtype=torch.float32)
        _lib.check(
            _lib.lib().imask_project(
                self.handle, factor, _ptr(u), u.numel(), _ptr(out), out.numel(), self.stream
            )
        )
        return out

    def backproject(self, y: torch.Tensor, factor: int, out: Optional[torch.Tensor] = None):
        n = self.geom.side // factor if self.geom.side % factor == 0 else 0
        if out is None:
            out = torch.empty(n * n, device=self.device, dtype=torch.float32)
        _lib.check(
            _lib.lib().imask_backproject(
                self.handle, factor, _ptr(y), y.numel(), _ptr(out), out.numel(), self.stream
            )
        )
        return out

    def sketch_forward(self, level: int, x: torch.Tensor, out: Optional[torch.Tensor] = None):
        if out is None:
            out = torch.empty(self.m_loc, device=self.device, dtype=torch.float32)
        _lib.check(
            _lib.lib().imask_sketch_forward(self.handle, level, _ptr(x), _ptr(out), self.stream)
        )
        return out

    def sketch_adjoint(self, level: int, y: torch.Tensor, out: Optional[torch.Tensor] = None):
        if out is None:
            out = torch.empty(self.geom.side ** 2, device=self.device, dtype=torch.float32)
        _lib.check(
            _lib.lib().imask_sketch_adjoint(self.handle, level, _ptr(y), _ptr(out), self.stream)
        )
        return out


_plan_cache: dict = {}
_plan_lock = threading.Lock()


def get_plan(geom: Geometry, r=1, probs=(1.0,), scale=1.0, angles=None, device=None) -> Plan:
    """Cached plan per (geometry, family, scale, angle set, device), like _projector_pair."""
    device = device or default_device()
    angles = _angle_list(geom, angles)
    key = (geom, int(r), tuple(float(p) for p in probs), float(scale), angles, str(device))
    with _plan_lock:
        plan = _plan_cache.get(key)
        if plan is None:
            plan = Plan(geom, r, probs, scale, device=device, angles=angles)
            _plan_cache[key] = plan
    return plan


@dataclass(frozen=True)
class ProjectorMeta:
    """What the fused solver needs to know about a projector LinOp."""

    geom: Geometry
    factor: int
    scale: float = 1.0
    angles: Optional[tuple] = None  # global angle indices of the rows (None: all)

    def scaled(self, alpha: float) -> "ProjectorMeta":
        return ProjectorMeta(self.geom, self.factor, self.scale * alpha, self.angles)

    @property
    def angle_list(self) -> tuple:
        return _angle_list(self.geom, self.angles)


def _projector_linop(geom: Geometry, factor: int, scale: float = 1.0, angles=None) -> LinOp:
    """R_f restricted to the rows of ``angles`` (all angles by default).

    The plan is resolved at first apply (after the caller has picked its CUDA device).
    """
    angles = None if angles is None else _int_tuple(angles)
    n_rows = geom.n_angles if angles is None else len(angles)
    low = geom.side // factor
    meta = ProjectorMeta(geom, factor, scale, angles)

    def plan():
        return get_plan(geom, scale=scale, angles=angles)

    return LinOp(
        low * low,
        n_rows * geom.n_detectors,
        lambda x: plan().project(to_device(x), factor),
        lambda y: plan().backproject(to_device(y), factor),
        meta,
    )


class _WidthProjector:
    """K of a grid of ``side`` pixels of width h = p/q, q = 2^k <= 64 (any
    multiple of 1/64; ctmodel.py:73-154 with
    pixel_width h), evaluated exactly by the unit-offset kernels through two
    identities of the chord matrix:
      ray_matrix(N, p/q, th, t) = (1/q) ray_matrix(N, p, th, q t)   (scale by q)
    and the offsets q t_j = q j - q (n-1)/2 are every q-th offset of a detector
    row of n' = q (n-1) + 1 unit-spaced bins. A grid of N pixels of width p is
    level factor p of the N p side plan, so the projection is that plan's
    factor-p projection of n' bins, every q-th bin kept, scaled by 1/q; the
    adjoint spreads the sinogram onto every q-th bin (zeros between) and
    backprojects. h = 1 is the plain plan (p = q = 1). The denominator is a
    power of two, so q t and the gridlines scale exactly in binary floating
    point and the reference's half-open tie rule picks the same pixels (with
    q = 3 it would not: ray_matrix itself decides those ties by rounding)."""

    MAX_DEN = 64

    def __init__(self, geom: Geometry, pixel_width: float):
        from fractions import Fraction

        h = float(pixel_width)
        if not h > 0.0 or not math.isfinite(h):
            raise ValueError("pixel_width must be positive")
        fr = Fraction(h)  # exact: a binary64 value is p / 2^k
        if fr.denominator > self.MAX_DEN:
            raise ValueError(f"pixel_width {h!r} is not a multiple of 1/{self.MAX_DEN}")
        self.geom, self.p, self.q = geom, fr.numerator, fr.denominator
        self.n_wide = self.q * (geom.n_detectors - 1) + 1
        self.wide = Geometry(geom.side * self.p, geom.n_angles, self.n_wide)

    def _plan(self) -> "Plan":
        return get_plan(self.wide, scale=1.0 / self.q)

    def project(self, x: torch.Tensor) -> torch.Tensor:
        g = self.geom
        full = self._plan().project(x, self.p)
        if self.q == 1:
            return full
        return full.reshape(g.n_angles, self.n_wide)[:, ::self.q].contiguous().reshape(-1)

    def backproject(self, y: torch.Tensor) -> torch.Tensor:
        g = self.geom
        if self.q > 1:
            wide = torch.zeros(g.n_angles, self.n_wide, device=y.device, dtype=torch.float32)
            wide[:, ::self.q] = y.reshape(g.n_angles, g.n_detectors)
            y = wide.reshape(-1)
        return self._plan().backproject(y, self.p)


def project(geom: Geometry, x, pixel_width: float = 1.0) -> torch.Tensor:
    """(n_angles, n_detectors) sinogram of an image (ctmodel.py:170-176); any
    pixel width that is a multiple of 1/64, through _WidthProjector."""
    t = to_device(x)
    if t.numel() != geom.side * geom.side:
        raise ValueError(f"image has {t.numel()} pixels, geometry expects {geom.side}^2")
    return _WidthProjector(geom, pixel_width).project(t).reshape(geom.n_angles, geom.n_detectors)


def backproject(geom: Geometry, y, pixel_width: float = 1.0) -> torch.Tensor:
    """Exact adjoint of project; (side, side) image (ctmodel.py:179-185)."""
    t = to_device(y)
    if t.numel() != geom.m:
        raise ValueError(f"sinogram has {t.numel()} bins, geometry expects {geom.m}")
    return _WidthProjector(geom, pixel_width).backproject(t).reshape(geom.side, geom.side)


def projector_op(geom: Geometry, pixel_width: float = 1.0, angles=None) -> LinOp:
    """Full-resolution forward model as a flat LinOp (ctmodel.py:188-191).

    ``angles`` (extension): global indices of the rows to keep, in row order
    (e.g. ``quad_subset`` for a sparse-view scan); all angles by default.
    """
    if float(pixel_width) != 1.0:
        if angles is not None:
            raise ValueError("angle subsets take the unit pixel width")
        wp = _WidthProjector(geom, pixel_width)
        return LinOp(geom.side * geom.side, geom.m, lambda x: wp.project(to_device(x)),
                     lambda y: wp.backproject(to_device(y)))
    return _projector_linop(geom, 1, angles=angles)


def coarse_projector(geom: Geometry, factor: int, angles=None) -> LinOp:
    """Forward model on the grid coarsened by ``factor`` (ctmodel.py:194-204)."""
    if geom.side % factor != 0:
        raise ValueError(f"side {geom.side} not divisible by factor {factor}")
    return _projector_linop(geom, factor, angles=angles)
