"""Seeded synthetic inputs for the BASELINE configs (host-side data generation).

The paper's XCAT/AAPM scans are not available offline, and the reference's
phantoms (flat / shepp-logan / square-insert, ctmodel.py:218-241) are not the
BASELINE's random-ellipse phantom, so both sides of every parity test and the
benchmark consume the same arrays generated here.

Phantom: sum of ``n_ellipses`` seeded ellipses sampled at pixel centres of
[-1,1]^2 with y increasing with row (the centre convention of
ctmodel.py:245-246), ellipse test (xr/a)^2 + (yr/b)^2 <= 1 as in
ctmodel.py:251-253, clipped to [0,1]. Draw order per ellipse, from
``numpy.random.default_rng(seed)``: cx, cy ~ U[-0.6,0.6]; a, b ~ U[0.05,0.4];
rotation ~ U[0,pi); intensity ~ U[0.1,1.0].

Noise: b = Kx + N(0, (kappa * max|Kx|)^2), ``default_rng(noise_seed)``,
one standard normal per bin in row-major sinogram order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def ellipse_phantom(side: int, seed: int = 0, n_ellipses: int = 10) -> np.ndarray:
    rng = np.random.default_rng(seed)
    coords = (np.arange(side) + 0.5) / side * 2.0 - 1.0
    xg, yg = np.meshgrid(coords, coords)
    img = np.zeros((side, side))
    for _ in range(n_ellipses):
        cx = rng.uniform(-0.6, 0.6)
        cy = rng.uniform(-0.6, 0.6)
        a = rng.uniform(0.05, 0.4)
        b = rng.uniform(0.05, 0.4)
        rot = rng.uniform(0.0, np.pi)
        val = rng.uniform(0.1, 1.0)
        c, s = np.cos(rot), np.sin(rot)
        xr = (xg - cx) * c + (yg - cy) * s
        yr = -(xg - cx) * s + (yg - cy) * c
        img[(xr / a) ** 2 + (yr / b) ** 2 <= 1.0] += val
    return np.clip(img, 0.0, 1.0)


def add_gaussian_noise(sino: np.ndarray, kappa: float, noise_seed: int = 1) -> np.ndarray:
    sino = np.asarray(sino, dtype=float)
    rng = np.random.default_rng(noise_seed)
    std = kappa * float(np.max(np.abs(sino)))
    return sino + std * rng.standard_normal(sino.shape)


@dataclass(frozen=True)
class CTConfig:
    """One BASELINE configuration (BASELINE.json `configs`)."""

    name: str
    side: int
    n_angles: int
    n_det: int
    levels: int
    kappa: float
    epochs: int
    mu_g: float = 1e-2

    @property
    def m(self) -> int:
        return self.n_angles * self.n_det

    @property
    def d(self) -> int:
        return self.side * self.side

    def iters_for_epochs(self) -> int:
        """Iterations whose expected cost is `epochs` (E[dcost] = 2 sum p_i / f_i, uniform p)."""
        r = self.levels
        per_iter = 2.0 * sum((1.0 / r) / 2 ** (r - i) for i in range(1, r + 1))
        return int(np.ceil(self.epochs / per_iter))


CONFIGS = {
    "A": CTConfig("A-128", 128, 180, 183, 3, 0.01, 20),
    "B": CTConfig("B-256", 256, 360, 363, 4, 0.02, 30),
    "C": CTConfig("C-512", 512, 720, 725, 5, 0.01, 40),
    "D": CTConfig("D-1024", 1024, 1440, 1449, 6, 0.01, 50),
    "E": CTConfig("E-2048-microbench", 2048, 2048, 2897, 7, 0.0, 0),
}
