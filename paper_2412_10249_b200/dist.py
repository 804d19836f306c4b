"""Angle-sharded multi-GPU ImaSk.

One process per GPU. Rank p owns a mirror-closed angle shard
(ctmodel.shard_angles): base angles a in 1..n/2 (block-cyclic groups of the
forward's eight-entry CTAs, contiguous runs on small angle sets) plus their
mirrors n - a (theta -> pi - theta), and angle 0 on rank 0, so every rank
runs the mirror-symmetric kernels; its rows of y, b, the psi table and
psi_sum live only there. Every rank draws the same level from the
counter-based RNG, backprojects its shard, and the coarse partial image is
summed with one NCCL all-reduce -- the only collective -- while the forward
projection of the shard runs on the compute stream; the image-side update is
then replicated on every rank (solvers._device_step).
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from . import ctmodel, linops, mrsketch, proxlib, solvers


def shard_projector(geom: ctmodel.Geometry, factor: int, rank: int, world: int,
                    scale: float = 1.0) -> linops.LinOp:
    """R_f on this rank's mirror-closed angle shard: domain (side/f)^2, range
    len(shard_angles) * n_det, rows in shard order."""
    return ctmodel._projector_linop(geom, factor, scale,
                                    ctmodel.shard_angles(geom.n_angles, rank, world))


def local_rows(geom: ctmodel.Geometry, b_full, rank: int, world: int) -> np.ndarray:
    """This rank's rows of a full (n_angles x n_det) sinogram, in shard order."""
    idx = np.asarray(ctmodel.shard_angles(geom.n_angles, rank, world), dtype=np.int64)
    return np.asarray(b_full).reshape(geom.n_angles, geom.n_detectors)[idx].ravel()


def make_sharded_problem(geom: ctmodel.Geometry, b_loc, family: mrsketch.SketchFamily,
                         mu_g: float, rank: int = 0, world: int = 1, group=None,
                         scale: float = 1.0) -> solvers.Problem:
    """Coarse-mode ridge problem on this rank's shard (b_loc = local_rows(b))."""
    K = shard_projector(geom, 1, rank, world, scale)
    return solvers.make_problem(
        K, b_loc, family, proxlib.ridge_fn(mu_g), proxlib.quadratic_conjugate_fn(b_loc),
        coarse_projector=lambda f: shard_projector(geom, f, rank, world, scale),
        shard=solvers.Shard(rank, world, group),
    )
