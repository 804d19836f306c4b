"""Float64 CPU oracle of the reference exact-chord projector (TEST INFRASTRUCTURE).

Restates `mrtomo.ctmodel` (reference `pkg/src/mrtomo/ctmodel.py`) for the
hot path: `Geometry.angles/offsets` (ctmodel.py:63-70), the exact ray/pixel
chord matrix `ray_matrix` (ctmodel.py:73-154), and the applies built on it:
`project` / `backproject` (ctmodel.py:170-185) and `coarse_projector`
(ctmodel.py:194-204: same detectors, grid side/f, pixel width f).

The reference builds a Siddon CSR matrix by sorting gridline crossings. The
restatement here evaluates the same chords per *row band* (or column band)
of the grid, which is algebraically identical and is the formulation the CUDA
kernels use: a non-horizontal ray crosses the band of one pixel row along a
segment of length h/|cos| whose x-extent is tau*h wide (tau = |sin|/|cos|);
the segment splits between at most two pixels of that row, with fractions
(1-g, g), g = clip(frac/tau - (1-tau)/(2 tau), 0, 1) where frac is the ray's
offset from the left pixel's centre in pixel units. Rows are swapped for
columns when |sin| > |cos|. Axis-parallel rays (cos or sin snapped to 0 below
1e-14, ctmodel.py:20,90-93) keep the reference's half-open tie rule: a ray on
a gridline belongs to the upper/right pixel, coord in [-half, half)
(ctmodel.py:99-114). Chords <= 1e-12*max(1,h) are dropped as in
ctmodel.py:21,133.

Pinned against the reference's own `ray_matrix` / `project` / `backproject`
outputs (tests/golden/, tests/test_oracle.py).
"""

from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np

AXIS_SNAP = 1e-14  # ctmodel.py:20
SEG_TOL = 1e-12  # ctmodel.py:21


def default_detectors(side: int) -> int:
    """ctmodel.py:54-57: ceil(sqrt(2) * side) bins cover the diagonal."""
    return math.ceil(math.sqrt(2.0 * side * side))


def angles(n_angles: int) -> np.ndarray:
    """theta_a = a * pi / n_angles (ctmodel.py:63-65)."""
    return np.arange(n_angles) * (np.pi / n_angles)


def offsets(n_det: int) -> np.ndarray:
    """Unit-pitch centred detector offsets t_j = j - (n_d-1)/2 (ctmodel.py:67-70)."""
    return np.arange(n_det, dtype=float) - (n_det - 1) / 2.0


def snapped_cos_sin(theta: float) -> tuple[float, float]:
    """cos/sin with the reference's 1e-14 snap to exact zero (ctmodel.py:88-93)."""
    c = math.cos(theta)
    s = math.sin(theta)
    if abs(c) < AXIS_SNAP:
        c = 0.0
    if abs(s) < AXIS_SNAP:
        s = 0.0
    return c, s


def angle_chords(side: int, h: float, c: float, s: float, t: np.ndarray):
    """All nonzero chords of one projection angle.

    Returns (ray, pixel, length) triplets: ray indexes ``t``, pixel is the
    row-major flat index on the side x side grid of width h.
    """
    n = int(side)
    half = n * h / 2.0
    n_d = t.size
    if c == 0.0 or s == 0.0:
        # axis-parallel rays cover one full pixel row/column (ctmodel.py:99-114)
        along_x = c == 0.0  # direction (-s, c): c == 0 -> ray runs along x
        coord = t * s if along_x else t * c
        line = np.floor((coord + half) / h).astype(np.int64)
        ok = (line >= 0) & (line < n) & (coord < half) & (coord >= -half)
        rays = np.nonzero(ok)[0]
        k = np.arange(n, dtype=np.int64)
        if along_x:
            pix = line[rays, None] * n + k[None, :]
        else:
            pix = k[None, :] * n + line[rays, None]
        return (
            np.repeat(rays, n),
            pix.ravel(),
            np.full(rays.size * n, float(h)),
        )
    # oblique: one chord pair per row band (|c| >= |s|) or column band
    row_family = abs(c) >= abs(s)
    centers = -half + (np.arange(n) + 0.5) * h
    if row_family:
        cross = (t[:, None] - centers[None, :] * s) / c  # x where ray meets row centre line
        tau = abs(s) / abs(c)
        w_band = h / abs(c)
    else:
        cross = (t[:, None] - centers[None, :] * c) / s  # y where ray meets column centre line
        tau = abs(c) / abs(s)
        w_band = h / abs(s)
    pos = (cross + half) / h - 0.5  # fractional index along the band
    lo = np.floor(pos)
    frac = pos - lo
    lo = lo.astype(np.int64)
    g = np.clip((frac - 0.5 * (1.0 - tau)) / tau, 0.0, 1.0)
    w_lo = w_band * (1.0 - g)
    w_hi = w_band * g
    band = np.broadcast_to(np.arange(n, dtype=np.int64)[None, :], pos.shape)
    ray = np.broadcast_to(np.arange(n_d, dtype=np.int64)[:, None], pos.shape)
    tol = SEG_TOL * max(1.0, h)
    out_r, out_p, out_w = [], [], []
    for idx, w in ((lo, w_lo), (lo + 1, w_hi)):
        keep = (w > tol) & (idx >= 0) & (idx < n)
        if row_family:
            pix = band[keep] * n + idx[keep]
        else:
            pix = idx[keep] * n + band[keep]
        out_r.append(ray[keep])
        out_p.append(pix)
        out_w.append(w[keep])
    return np.concatenate(out_r), np.concatenate(out_p), np.concatenate(out_w)


class ProjectorOracle:
    """Matrix-free float64 projector on the (side/f)^2 grid, pixel width f.

    ``angle_idx`` restricts the scan to a subset (or slab) of the geometry's
    angles -- the sampled-angle oracle used at 1024^2 / 2048^2.
    Rows of the sinogram follow ``angle_idx`` order.
    """

    def __init__(
        self,
        side: int,
        n_angles: int,
        n_det: Optional[int] = None,
        factor: int = 1,
        angle_idx: Optional[Sequence[int]] = None,
        scale: float = 1.0,
    ):
        if side % factor != 0:
            raise ValueError(f"side {side} not divisible by factor {factor}")
        self.side = side
        self.n_angles = n_angles
        self.n_det = default_detectors(side) if n_det is None else int(n_det)
        self.factor = factor
        self.low = side // factor
        self.h = float(factor)
        self.scale = float(scale)
        self.angle_idx = (
            np.arange(n_angles) if angle_idx is None else np.asarray(angle_idx, dtype=np.int64)
        )
        th = angles(n_angles)
        self.t = offsets(self.n_det)
        self._chords = []
        for a in self.angle_idx:
            c, s = snapped_cos_sin(float(th[a]))
            self._chords.append(angle_chords(self.low, self.h, c, s, self.t))
        self._csr = None
        self._csr_t = None

    def csr_pair(self):
        """(A, A^T) in CSR, cached like ctmodel._projector_pair (ctmodel.py:157-167)."""
        if self._csr is None:
            self._csr = self.to_csr()
            self._csr_t = self._csr.T.tocsr()
        return self._csr, self._csr_t

    def set_threads(self, pool, n_threads: int) -> None:
        """Multi-core CPU baseline: both CSR matvecs split into `n_threads` row
        blocks run on `pool` (scipy's csr_matvec releases the GIL). Each block
        writes its own output rows, so results equal the one-core product."""
        a, at = self.csr_pair()
        # small operators stay on one core: a thread hand-off costs more than the product
        n_threads = int(min(n_threads, max(1, a.nnz // 100_000)))

        def blocks(m):
            cuts = np.linspace(0, m.shape[0], n_threads + 1).astype(np.int64)
            return [m[lo:hi] for lo, hi in zip(cuts[:-1], cuts[1:]) if hi > lo]

        self._pool = pool
        self._blocks = (blocks(a), blocks(at))

    def _matvec(self, which: int, v: np.ndarray) -> np.ndarray:
        if getattr(self, "_pool", None) is None:
            return (self._csr, self._csr_t)[which] @ v
        return np.concatenate(list(self._pool.map(lambda blk: blk @ v, self._blocks[which])))

    @property
    def domain_dim(self) -> int:
        return self.low * self.low

    @property
    def range_dim(self) -> int:
        return len(self.angle_idx) * self.n_det

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = np.asarray(x, dtype=float).ravel()
        if x.size != self.domain_dim:
            raise ValueError(f"image has {x.size} pixels, expected {self.domain_dim}")
        if self._csr is not None:
            return self._matvec(0, x)
        out = np.empty((len(self.angle_idx), self.n_det))
        for k, (ray, pix, w) in enumerate(self._chords):
            out[k] = np.bincount(ray, weights=w * x[pix], minlength=self.n_det)
        return (self.scale * out).ravel()

    def adjoint_apply(self, y: np.ndarray) -> np.ndarray:
        if self._csr is not None:
            return self._matvec(1, np.asarray(y, dtype=float).ravel())
        y = np.asarray(y, dtype=float).reshape(len(self.angle_idx), self.n_det)
        img = np.zeros(self.domain_dim)
        for k, (ray, pix, w) in enumerate(self._chords):
            img += np.bincount(pix, weights=w * y[k][ray], minlength=self.domain_dim)
        return self.scale * img

    def nnz(self) -> int:
        return int(sum(r.size for r, _, _ in self._chords))

    def to_csr(self):
        """The reference's CSR operator (float64 values, int32 indices) for the CPU baseline."""
        from scipy import sparse

        rows, cols, vals = [], [], []
        for k, (ray, pix, w) in enumerate(self._chords):
            rows.append(ray + k * self.n_det)
            cols.append(pix)
            vals.append(self.scale * w)
        mat = sparse.coo_matrix(
            (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
            shape=(self.range_dim, self.domain_dim),
        )
        return mat.tocsr()


def project(side, n_angles, n_det, x, factor=1, angle_idx=None, scale=1.0):
    return ProjectorOracle(side, n_angles, n_det, factor, angle_idx, scale).apply(x)


def backproject(side, n_angles, n_det, y, factor=1, angle_idx=None, scale=1.0):
    return ProjectorOracle(side, n_angles, n_det, factor, angle_idx, scale).adjoint_apply(y)
