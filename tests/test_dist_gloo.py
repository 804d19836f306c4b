"""Angle-sharded multi-rank logic on CPU (world_size 2, gloo).

The B200 path shards projection angles into mirror-closed shards
(ctmodel.shard_angles: a and n - a on the same rank, so every rank runs the
symmetric kernels): each rank backprojects its shard and the partial images
are summed by one all-reduce. These tests check, with the
float64 oracle standing in for the device kernels and the product's own
sharding helpers (shard_angles, dist.local_rows), that shard-partial
backprojections all-reduce to the full backprojection, that shard forward
projections scatter back to the full sinogram, that every rank draws the
identical level schedule from the C library, and that a sharded ImaSk
iteration equals the unsharded one.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ct_oracle, sketch_oracle
from paper_2412_10249_b200 import dist as dist_mod
from paper_2412_10249_b200.ctmodel import Geometry, shard_angles


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _scatter_rows(part, idx, n_angles, n_det):
    """This rank's rows placed into a zero full sinogram (summed over ranks)."""
    full = np.zeros((n_angles, n_det))
    full[np.asarray(idx)] = np.asarray(part).reshape(len(idx), n_det)
    return torch.from_numpy(full.ravel())


def _worker(rank, world, port, q, n_angles):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_10249_b200.solvers import draw_levels

        side, n_det, r = 32, 47, 3
        probs = [1 / 3] * 3
        idx = shard_angles(n_angles, rank, world)
        rng = np.random.default_rng(5)
        x = rng.standard_normal(side * side)
        y = rng.standard_normal(n_angles * n_det)
        y_loc = dist_mod.local_rows(Geometry(side, n_angles, n_det), y, rank, world)
        res = {}
        for f in (1, 2, 4):
            op = ct_oracle.ProjectorOracle(side, n_angles, n_det, f, angle_idx=idx)
            bp = torch.from_numpy(op.adjoint_apply(y_loc))
            dist.all_reduce(bp)
            res[f"bp{f}"] = bp.numpy()
            xl = sketch_oracle.decimate(x.reshape(side, side), f).ravel()
            full = _scatter_rows(op.apply(xl), idx, n_angles, n_det)
            dist.all_reduce(full)
            res[f"fw{f}"] = full.numpy()
        sched = torch.from_numpy(draw_levels(99, 0, 256, np.cumsum(probs)).astype(np.int64))
        all_s = [torch.zeros_like(sched) for _ in range(world)]
        dist.all_gather(all_s, sched)
        res["sched_equal"] = all(torch.equal(all_s[0], s) for s in all_s)
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("n_angles", [30, 31])
def test_sharded_projections_world2(n_angles):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, n_angles))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    side, n_det = 32, 47
    rng = np.random.default_rng(5)
    x = rng.standard_normal(side * side)
    y = rng.standard_normal(n_angles * n_det)
    for f in (1, 2, 4):
        op = ct_oracle.ProjectorOracle(side, n_angles, n_det, f)
        assert np.allclose(res[f"bp{f}"], op.adjoint_apply(y), rtol=0, atol=1e-10)
        xl = sketch_oracle.decimate(x.reshape(side, side), f).ravel()
        assert np.allclose(res[f"fw{f}"], op.apply(xl), rtol=0, atol=1e-10)
    assert res["sched_equal"]


def _step_worker(rank, world, port, q):
    """A sharded ImaSk iteration: local psi/y slab updates + all-reduced phi update."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import solver_oracle as so

        side, n_angles, n_det, probs = 32, 30, 47, [1 / 3] * 3
        idx = shard_angles(n_angles, rank, world)
        ops = so.SketchedCT(side, n_angles, n_det, probs, angle_idx=idx)
        rng = np.random.default_rng(8)
        b_full = rng.standard_normal(n_angles * n_det)
        b = dist_mod.local_rows(Geometry(side, n_angles, n_det), b_full, rank, world)
        st = so.init_state(ops, seed=4)
        sigma, mu, mu_g = 1e-3, 1e-2, 1e-2
        cum = np.cumsum(probs)
        for _ in range(12):
            i = so.draw_level(st.seed, st.k, cum)
            phi_new = torch.from_numpy(ops.adjoint_apply(i, st.y))
            dist.all_reduce(phi_new)  # compensation / prolongation are linear: reduce after
            phi_new = phi_new.numpy()
            psi_new = ops.apply(i, st.x)
            xi = (phi_new - st.phi[i]) + st.phi_sum
            zeta = (psi_new - st.psi[i]) + st.psi_sum
            st.phi_sum = st.phi_sum + probs[i] * (phi_new - st.phi[i])
            st.psi_sum = st.psi_sum + probs[i] * (psi_new - st.psi[i])
            st.phi[i], st.psi[i] = phi_new, psi_new
            s = sigma / mu
            st.x = (st.x - s * xi) / (1 + s * mu_g)
            st.y = ((st.y + sigma * zeta) - sigma * b) / (1 + sigma)
            st.k += 1
        y_full = _scatter_rows(st.y, idx, n_angles, n_det)
        dist.all_reduce(y_full)
        if rank == 0:
            q.put({"x": st.x, "y": y_full.numpy()})
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_iterations_match_single_rank():
    from oracle import solver_oracle as so

    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_step_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    side, n_angles, n_det, probs = 32, 30, 47, [1 / 3] * 3
    ops = so.SketchedCT(side, n_angles, n_det, probs)
    b = np.random.default_rng(8).standard_normal(n_angles * n_det)
    st = so.init_state(ops, seed=4)
    for _ in range(12):
        so.sketch_step(st, ops, b, 1e-3, 1e-2, 1e-2)
    assert np.allclose(res["x"], st.x, rtol=0, atol=1e-9 * np.abs(st.x).max())
    assert np.allclose(res["y"], st.y, rtol=0, atol=1e-9 * np.abs(st.y).max())
