"""Angle-sharded multi-GPU ImaSk.

One process per GPU. Rank p owns the contiguous angle slab
[p*n/P, (p+1)*n/P) (extra angles to the first ranks): its rows of y, b, the
psi table and psi_sum live only there. Every rank draws the same level from
the counter-based RNG, backprojects its slab, and the coarse partial image
is summed with one NCCL all-reduce -- the only collective -- while the
forward projection of the slab runs on the compute stream; the image-side
update is then replicated on every rank (solvers._device_step).
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from . import ctmodel, linops, mrsketch, proxlib, solvers


def slab_projector(geom: ctmodel.Geometry, factor: int, rank: int, world: int,
                   scale: float = 1.0) -> linops.LinOp:
    """R_f on this rank's angle slab: domain (side/f)^2, range slab_angles * n_det."""
    begin, end = ctmodel.slab_bounds(geom.n_angles, rank, world)
    return ctmodel._projector_linop(geom, factor, scale, begin, end)


def local_rows(geom: ctmodel.Geometry, b_full, rank: int, world: int) -> np.ndarray:
    """This rank's rows of a full (n_angles x n_det) sinogram."""
    begin, end = ctmodel.slab_bounds(geom.n_angles, rank, world)
    return np.asarray(b_full).reshape(geom.n_angles, geom.n_detectors)[begin:end].ravel()


def make_sharded_problem(geom: ctmodel.Geometry, b_loc, family: mrsketch.SketchFamily,
                         mu_g: float, rank: int = 0, world: int = 1, group=None,
                         scale: float = 1.0) -> solvers.Problem:
    """Coarse-mode ridge problem on this rank's slab (b_loc = local_rows(b))."""
    K = slab_projector(geom, 1, rank, world, scale)
    return solvers.make_problem(
        K, b_loc, family, proxlib.ridge_fn(mu_g), proxlib.quadratic_conjugate_fn(b_loc),
        coarse_projector=lambda f: slab_projector(geom, f, rank, world, scale),
        shard=solvers.Shard(rank, world, group),
    )
