"""Angle-sharded multi-rank logic on CPU (world_size 2, gloo).

The B200 path shards projection angles: each rank backprojects its slab and
the partial images are summed by one all-reduce. These tests
check, with the float64 oracle standing in for the device kernels, that
slab-partial backprojections all-reduce to the full backprojection, that
slab forward projections concatenate to the full sinogram, that every rank
draws the identical level schedule from the C library, and that a sharded
ImaSk iteration equals the unsharded one.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ct_oracle, sketch_oracle
from paper_2412_10249_b200.ctmodel import slab_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_10249_b200.solvers import draw_levels

        side, n_angles, n_det, r = 32, 30, 47, 3
        probs = [1 / 3] * 3
        begin, end = slab_bounds(n_angles, rank, world)
        rng = np.random.default_rng(5)
        x = rng.standard_normal(side * side)
        y = rng.standard_normal(n_angles * n_det)
        y_loc = y.reshape(n_angles, n_det)[begin:end].ravel()
        res = {}
        for f in (1, 2, 4):
            op = ct_oracle.ProjectorOracle(side, n_angles, n_det, f, angle_idx=range(begin, end))
            bp = torch.from_numpy(op.adjoint_apply(y_loc))
            dist.all_reduce(bp)
            res[f"bp{f}"] = bp.numpy()
            xl = sketch_oracle.decimate(x.reshape(side, side), f).ravel()
            part = torch.from_numpy(op.apply(xl))
            parts = [torch.zeros(n_det * (e - b), dtype=part.dtype)
                     for b, e in (slab_bounds(n_angles, k, world) for k in range(world))]
            dist.all_gather(parts, part)
            res[f"fw{f}"] = torch.cat(parts).numpy()
        sched = torch.from_numpy(draw_levels(99, 0, 256, np.cumsum(probs)).astype(np.int64))
        all_s = [torch.zeros_like(sched) for _ in range(world)]
        dist.all_gather(all_s, sched)
        res["sched_equal"] = all(torch.equal(all_s[0], s) for s in all_s)
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_projections_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    side, n_angles, n_det = 32, 30, 47
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
        begin, end = slab_bounds(n_angles, rank, world)
        ops = so.SketchedCT(side, n_angles, n_det, probs, angle_idx=range(begin, end))
        rng = np.random.default_rng(8)
        b_full = rng.standard_normal(n_angles * n_det)
        b = b_full.reshape(n_angles, n_det)[begin:end].ravel()
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
        ys = [torch.zeros(n_det * (e - bb), dtype=torch.float64)
              for bb, e in (slab_bounds(n_angles, k, world) for k in range(world))]
        dist.all_gather(ys, torch.from_numpy(st.y))
        if rank == 0:
            q.put({"x": st.x, "y": torch.cat(ys).numpy()})
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
