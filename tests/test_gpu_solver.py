"""Parity of the fused sketched SAGA iteration (kernel 4 + engine) with the reference.

Budget (north star): the level sequence bit-exact; iterates after a fixed
iteration count within 1e-3 relative L2 of the reference on the same inputs,
sigma, mu and seed.
"""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import ct_oracle, solver_oracle as so
from paper_2412_10249_b200 import ctmodel, linops, mrsketch, proxlib, solvers
from paper_2412_10249_b200.synth import CONFIGS

pytestmark = pytest.mark.gpu


def host(t):
    torch.cuda.synchronize()
    return t.double().cpu().numpy().ravel()


def build(side, na, nd, probs, b, mu_g=1e-2, scale=1.0):
    geom = ctmodel.Geometry(side, na, nd)
    K = ctmodel.projector_op(geom)
    coarse = lambda f: ctmodel.coarse_projector(geom, f)
    if scale != 1.0:
        K = linops.scale(K, scale)
        coarse = lambda f, c=coarse: linops.scale(c(f), scale)
    fam = mrsketch.make_family(len(probs), side, probs, mode="coarse")
    prob = solvers.make_problem(K, b, fam, proxlib.ridge_fn(mu_g),
                                proxlib.quadratic_conjugate_fn(b), coarse_projector=coarse)
    assert prob.engine is not None
    return prob


def test_trajectory_config_A(g_solver_A):
    cfg = CONFIGS["A"]
    b = g_solver_A["b"]
    prob = build(cfg.side, cfg.n_angles, cfg.n_det, [1 / 3] * 3, b, cfg.mu_g)
    sigma, mu = float(g_solver_A["sigma"]), float(g_solver_A["mu"])
    st = solvers.init_state(prob, seed=int(g_solver_A["seed"]))
    levels = []
    for k in range(1, 201):
        solvers.sketch_step(st, prob, sigma, mu)
        levels.append(st.last_level)
        if k in (18, 200):
            assert rel_l2(host(st.x), g_solver_A[f"x_{k}"]) <= 1e-3, k
            assert rel_l2(host(st.y), g_solver_A[f"y_{k}"]) <= 1e-3, k
            assert rel_l2(host(st.phi_sum), g_solver_A[f"phi_sum_{k}"]) <= 1e-3, k
            assert rel_l2(host(st.psi_sum), g_solver_A[f"psi_sum_{k}"]) <= 1e-3, k
            assert st.cost == float(g_solver_A[f"cost_{k}"])
    assert levels == g_solver_A["levels"].astype(int).tolist()


def test_single_steps_tables_vs_oracle():
    side, na, nd, probs = 64, 90, 91, [0.3, 0.3, 0.2, 0.2]
    orc = so.SketchedCT(side, na, nd, probs)
    rng = np.random.default_rng(0)
    b = orc.proj[1].apply(rng.random(side * side))
    prob = build(side, na, nd, probs, b)
    st = solvers.init_state(prob, seed=5)
    ost = so.init_state(orc, seed=5)
    fam = prob.family
    for _ in range(6):
        solvers.sketch_step(st, prob, 2e-4, 1e-2)
        so.sketch_step(ost, orc, b, 2e-4, 1e-2, 1e-2)
        assert st.last_level == ost.last_level
        i = st.last_level - 1
        assert rel_l2(host(st.phi_full(i, fam)), ost.phi[i]) <= 1e-4
        assert rel_l2(host(st.psi[i]), ost.psi[i]) <= 1e-4
        assert rel_l2(host(st.x), ost.x) <= 1e-4
        assert rel_l2(host(st.y), ost.y) <= 1e-4


@pytest.mark.parametrize("graphs", [True, False])
def test_double_buffered_dual_matches_in_place(graphs):
    """y_next (forward concurrent with the adjoint on a side stream) and the
    in-place update give the same iterates, through graphs and eager calls."""
    side, na, nd, probs = 64, 90, 91, [0.3, 0.3, 0.2, 0.2]
    orc = so.SketchedCT(side, na, nd, probs)
    b = orc.proj[1].apply(np.random.default_rng(4).random(side * side))
    prob = build(side, na, nd, probs, b)
    prob.engine.use_graphs = graphs
    st_db = solvers.init_state(prob, seed=3)
    st_ip = solvers.init_state(prob, seed=3)
    st_ip.y_alt = None
    for _ in range(12):
        solvers.sketch_step(st_db, prob, 2e-4, 1e-2)
        solvers.sketch_step(st_ip, prob, 2e-4, 1e-2)
    prob.engine.release_graphs()
    for a, c in ((st_db.x, st_ip.x), (st_db.y, st_ip.y), (st_db.phi_sum, st_ip.phi_sum),
                 (st_db.psi_sum, st_ip.psi_sum)):
        assert np.array_equal(host(a), host(c))


@pytest.mark.parametrize("world,key", [(2, None), (3, None), (8, "D")])
def test_sharded_phases_match_single_gpu(world, key):
    """The multi-GPU step emulated in one process: every rank's
    mirror-closed shard runs step_adjoint on its own plan, the partial coarse
    backprojections are summed (the NCCL all-reduce), then step_forward and
    step_image; x stays identical across ranks and matches the single-GPU run."""
    import ctypes

    from paper_2412_10249_b200 import _lib
    from paper_2412_10249_b200 import dist as dist_mod

    if key is None:
        side, na, nd, probs, mu_g = 64, 90, 91, [0.3, 0.3, 0.2, 0.2], 1e-2
        orc = so.SketchedCT(side, na, nd, probs)
        b = orc.proj[1].apply(np.random.default_rng(6).random(side * side))
    else:
        # the benchmarked configuration on 8 ranks: block-cyclic quad shards, the TMA
        # kernels and fused staging on every shard
        cfg = CONFIGS[key]
        side, na, nd, mu_g = cfg.side, cfg.n_angles, cfg.n_det, cfg.mu_g
        probs = [1.0 / cfg.levels] * cfg.levels
        b = np.random.default_rng(6).random(na * nd) * side
    geom = ctmodel.Geometry(side, na, nd)
    fam = mrsketch.make_family(len(probs), side, probs, mode="coarse")
    single = dist_mod.make_sharded_problem(geom, b, fam, mu_g)
    st1 = solvers.init_state(single, seed=2)
    ranks = []
    for rank in range(world):
        pr = dist_mod.make_sharded_problem(geom, dist_mod.local_rows(geom, b, rank, world), fam,
                                           mu_g, rank, world)
        assert pr.engine.plan.symmetric
        ranks.append((pr, solvers.init_state(pr, seed=2)))
    prm = solvers._params(2e-4, 1e-2, mu_g)
    L = _lib.lib()
    sched = (solvers.draw_levels(2, 0, 10, single.cum_probs) if key is None
             else list(range(len(probs))) * 2)
    for lv in (int(v) for v in sched):
        solvers._device_step(single.engine, st1, lv, prm)
        n = (side // single.engine.plan.factors[lv]) ** 2
        for pr, st in ranks:
            _lib.check(L.imask_step_adjoint(pr.engine.plan.handle,
                                            ctypes.byref(st.c_state(pr.engine.b)), lv,
                                            pr.engine.plan.stream))
        total = sum(st.bp[:n].clone() for _, st in ranks)
        for pr, st in ranks:
            st.bp[:n].copy_(total)
            cst = ctypes.byref(st.c_state(pr.engine.b))
            _lib.check(L.imask_step_forward(pr.engine.plan.handle, cst, lv, ctypes.byref(prm),
                                            pr.engine.plan.stream))
            _lib.check(L.imask_step_image(pr.engine.plan.handle, cst, lv, ctypes.byref(prm),
                                          pr.engine.plan.stream))
            st.swap_dual()
    x0 = host(ranks[0][1].x)
    for _, st in ranks[1:]:
        assert np.array_equal(host(st.x), x0)
    assert rel_l2(x0, host(st1.x)) <= 1e-5
    y1 = host(st1.y).reshape(na, nd)
    for rank, (_, st) in enumerate(ranks):
        idx = list(ctmodel.shard_angles(na, rank, world))
        assert rel_l2(host(st.y).reshape(len(idx), nd), y1[idx]) <= 1e-5


@pytest.mark.parametrize("side,na,nd,r", [(64, 90, 91, 3), (256, 360, 363, 4)])
def test_folded_plane_reduction_matches_explicit(side, na, nd, r):
    """The single-GPU step lets the image-side kernel sum the adjoint's split
    planes (in the reduce kernels' order); the phase entry points reduce them
    into bp first. Both give bit-identical iterates at every level, including
    the warp-tree order of many planes (256^2 / 360 angles, f = 8)."""
    import ctypes

    from paper_2412_10249_b200 import _lib
    from paper_2412_10249_b200 import dist as dist_mod

    geom = ctmodel.Geometry(side, na, nd)
    probs = [1.0 / r] * r
    b = np.random.default_rng(8).random(geom.m)
    fam = mrsketch.make_family(r, side, probs, mode="coarse")
    pr = dist_mod.make_sharded_problem(geom, b, fam, 1e-2)
    st_f, st_p = solvers.init_state(pr, seed=4), solvers.init_state(pr, seed=4)
    prm = solvers._params(2e-4, 1e-2, 1e-2)
    L = _lib.lib()
    h, stream = pr.engine.plan.handle, pr.engine.plan.stream
    for lv in list(range(r)) * 2:
        solvers._device_step(pr.engine, st_f, lv, prm)
        cst = ctypes.byref(st_p.c_state(pr.engine.b))
        _lib.check(L.imask_step_adjoint(h, cst, lv, stream))
        _lib.check(L.imask_step_forward(h, cst, lv, ctypes.byref(prm), stream))
        _lib.check(L.imask_step_image(h, cst, lv, ctypes.byref(prm), stream))
        st_p.swap_dual()
    torch.cuda.synchronize()
    for a, c in ((st_f.x, st_p.x), (st_f.y, st_p.y), (st_f.phi_sum, st_p.phi_sum),
                 (st_f.phi_tab, st_p.phi_tab)):
        assert np.array_equal(host(a), host(c))


@pytest.mark.parametrize("side,na,nd", [(64, 90, 91), (256, 180, 363)])
def test_sharded_device_step_stream_ordering(monkeypatch, side, na, nd):
    """solvers._device_step's multi-GPU branch (forward chain on a side stream,
    adjoint + all-reduce on the main stream; at 256^2 the large levels order the
    adjoint behind the forward's staging, imask_step_wait_staging) on rank 0 of
    a 2-rank shard, with the collective stubbed out, equals the three phases run
    back to back."""
    import ctypes

    from paper_2412_10249_b200 import _lib
    from paper_2412_10249_b200 import dist as dist_mod

    class _Done:
        def wait(self):
            pass

    monkeypatch.setattr(solvers, "_allreduce", lambda eng, t, async_op=False: _Done())
    probs, mu_g = [0.3, 0.3, 0.2, 0.2], 1e-2
    geom = ctmodel.Geometry(side, na, nd)
    b = np.random.default_rng(7).standard_normal(geom.m)
    fam = mrsketch.make_family(4, side, probs, mode="coarse")
    pr = dist_mod.make_sharded_problem(geom, dist_mod.local_rows(geom, b, 0, 2), fam, mu_g, 0, 2)
    st_a = solvers.init_state(pr, seed=9)
    st_b = solvers.init_state(pr, seed=9)
    st_b.y_alt = None  # in-place reference: phases strictly in order
    prm = solvers._params(2e-4, 1e-2, mu_g)
    L = _lib.lib()
    h, s = pr.engine.plan.handle, pr.engine.plan.stream
    for lv in (3, 0, 2, 1, 3, 3, 0):
        solvers._device_step(pr.engine, st_a, lv, prm)
        cst = ctypes.byref(st_b.c_state(pr.engine.b))
        _lib.check(L.imask_step_adjoint(h, cst, lv, s))
        _lib.check(L.imask_step_forward(h, cst, lv, ctypes.byref(prm), s))
        _lib.check(L.imask_step_image(h, cst, lv, ctypes.byref(prm), s))
    for a, c in ((st_a.x, st_b.x), (st_a.y, st_b.y), (st_a.phi_sum, st_b.phi_sum),
                 (st_a.psi_sum, st_b.psi_sum)):
        assert np.array_equal(host(a), host(c))


def test_graphs_retargeted_across_solves():
    """A second solve on the same problem reuses the cached step graphs
    (re-targeted to the new state's buffers when they differ) and reproduces
    the first solve bit for bit; so does an eager run."""
    side, na, nd, probs = 64, 90, 91, [0.3, 0.3, 0.2, 0.2]
    orc = so.SketchedCT(side, na, nd, probs)
    b = orc.proj[1].apply(np.random.default_rng(9).random(side * side))
    prob = build(side, na, nd, probs, b)
    n0 = len(prob.engine._graphs)  # the cache lives with the (shared) plan
    rep1 = solvers.run(prob, "sketch", 2e-4, 1e-2, 25, record_every=5, seed=4)
    n_graphs = len(prob.engine._graphs)
    assert n0 < n_graphs <= n0 + 2 * 4
    keep = rep1.x.clone()  # hold the first state's x so the second gets new buffers
    rep2 = solvers.run(prob, "sketch", 2e-4, 1e-2, 25, record_every=5, seed=4)
    assert len(prob.engine._graphs) == n_graphs
    assert np.array_equal(host(rep2.x), host(keep))
    prob.engine.use_graphs = False
    rep3 = solvers.run(prob, "sketch", 2e-4, 1e-2, 25, record_every=5, seed=4)
    assert np.array_equal(host(rep3.x), host(keep))
    assert [r[:3] for r in rep1.rows] == [r[:3] for r in rep2.rows] == [r[:3] for r in rep3.rows]


def test_resum_matches_direct_sums():
    side, na, nd, probs = 32, 36, 47, [0.3, 0.3, 0.2, 0.2]
    orc = so.SketchedCT(side, na, nd, probs)
    b = orc.proj[1].apply(np.random.default_rng(1).random(side * side))
    prob = build(side, na, nd, probs, b)
    st = solvers.init_state(prob, seed=8, resum_every=7)
    for _ in range(30):
        solvers.sketch_step(st, prob, 1e-3, 1e-2)
    direct_phi = sum(probs[i] * st.phi_full(i, prob.family).double() for i in range(4))
    direct_psi = sum(probs[i] * st.psi[i].double() for i in range(4))
    assert rel_l2(host(st.phi_sum), host(direct_phi)) <= 1e-5
    assert rel_l2(host(st.psi_sum), host(direct_psi)) <= 1e-5


def test_cost_ledger_and_run_report():
    side, na, nd, probs = 32, 36, 47, [0.25] * 4
    orc = so.SketchedCT(side, na, nd, probs)
    x_true = np.random.default_rng(2).random(side * side)
    b = orc.proj[1].apply(x_true)
    prob = build(side, na, nd, probs, b)
    rep = solvers.run(prob, "sketch", 1e-3, 1e-2, 50, record_every=10, seed=1, x_ref=x_true)
    assert [row[0] for row in rep.rows] == [0, 10, 20, 30, 40, 50]
    sched = so.level_schedule(1, 0, 50, probs)
    expected = 0.0
    for i in sched:
        expected += 2.0 * orc.fraction(int(i))
    assert rep.rows[-1][1] == expected
    assert rep.rows[-1][2] == int(sched[-1]) + 1
    ost = so.init_state(orc, seed=1)
    for _ in range(50):
        so.sketch_step(ost, orc, b, 1e-3, 1e-2, 1e-2)
    assert rel_l2(host(rep.x), ost.x) <= 1e-3
    rel_ref = float(np.dot(ost.x - x_true, ost.x - x_true) / np.dot(x_true, x_true))
    assert abs(rep.rows[-1][3] - rel_ref) <= 1e-3 * rel_ref
    # device-recorded rows: psnr as _metrics computes it, time stamps in order
    import torch
    x_t = torch.as_tensor(x_true, dtype=torch.float32, device=rep.x.device)
    assert abs(rep.rows[-1][4] - solvers.psnr(rep.x, x_t)) <= 1e-9 * abs(rep.rows[-1][4]) + 1e-9
    secs = [row[5] for row in rep.rows]
    assert all(b >= a for a, b in zip(secs, secs[1:]))
    assert rep.to_csv().startswith("k,cost,level,rel_dist,psnr,seconds\n0,0,0,")


def test_fixed_point_with_exact_memory():
    """test_solvers.py:121-131 on the device: the saddle point is stationary."""
    side, na, nd, probs, mu_g = 16, 20, 23, [0.25] * 4, 1.0
    orc = ct_oracle.ProjectorOracle(side, na, nd)
    Kd = orc.to_csr().toarray()
    b = Kd @ np.random.default_rng(3).random(side * side)
    x_star = np.linalg.solve(Kd.T @ Kd + mu_g * np.eye(side * side), Kd.T @ b)
    y_star = Kd @ x_star - b
    prob = build(side, na, nd, probs, b, mu_g=mu_g)
    st = solvers.init_state(prob, seed=5, x0=x_star, y0=y_star, exact_memory=True)
    scale_ref = max(np.linalg.norm(x_star), np.linalg.norm(y_star))
    for _ in range(8):
        solvers.sketch_step(st, prob, 2e-3, mu_g)
        assert np.linalg.norm(host(st.x) - x_star) <= 1e-5 * scale_ref
        assert np.linalg.norm(host(st.y) - y_star) <= 1e-5 * scale_ref


def test_normalised_operator_scale():
    side, na, nd, probs = 32, 36, 47, [1 / 3] * 3
    alpha = 1.0 / 37.5
    orc = so.SketchedCT(side, na, nd, probs, scale=alpha)
    b = orc.proj[1].apply(np.random.default_rng(6).random(side * side))
    prob = build(side, na, nd, probs, b, scale=alpha)
    st = solvers.init_state(prob, seed=2)
    ost = so.init_state(orc, seed=2)
    for _ in range(20):
        solvers.sketch_step(st, prob, 0.05, 1e-2)
        so.sketch_step(ost, orc, b, 0.05, 1e-2, 1e-2)
    assert rel_l2(host(st.x), ost.x) <= 1e-3
    assert rel_l2(host(st.y), ost.y) <= 1e-3


def test_long_run_config_B_levels_and_iterates():
    """Config B (r = 4) over 120 iterations at an empirically stable sigma."""
    cfg = CONFIGS["B"]
    probs = [0.25] * 4
    orc = so.SketchedCT(cfg.side, cfg.n_angles, cfg.n_det, probs)
    from paper_2412_10249_b200.synth import add_gaussian_noise, ellipse_phantom

    x_true = ellipse_phantom(cfg.side, 0).ravel()
    b = add_gaussian_noise(orc.proj[1].apply(x_true), cfg.kappa, 1)
    prob = build(cfg.side, cfg.n_angles, cfg.n_det, probs, b, cfg.mu_g)
    st = solvers.init_state(prob, seed=21)
    ost = so.init_state(orc, seed=21)
    for _ in range(120):
        solvers.sketch_step(st, prob, 1e-5, cfg.mu_g)
        so.sketch_step(ost, orc, b, 1e-5, cfg.mu_g, cfg.mu_g)
        assert st.last_level == ost.last_level
    assert rel_l2(host(st.x), ost.x) <= 1e-3
    assert rel_l2(host(st.y), ost.y) <= 1e-3


def test_rejects_bad_arguments():
    geom = ctmodel.Geometry(16, 20, 23)
    K = ctmodel.projector_op(geom)
    fam = mrsketch.make_family(2, 16, [0.5, 0.5], mode="exact")
    b = np.zeros(geom.m)
    prob = solvers.make_problem(K, b, fam, proxlib.ridge_fn(1.0), proxlib.quadratic_conjugate_fn(b))
    assert prob.engine is None  # exact mode: the generic device path (test_gpu_dropin.py)
    assert solvers.init_state(prob).phi_tab is None
    fam = mrsketch.make_family(2, 16, [0.5, 0.5], mode="coarse")
    with pytest.raises(ValueError, match="coarse_projector factory"):
        solvers.make_problem(K, b, fam, proxlib.ridge_fn(1.0), proxlib.quadratic_conjugate_fn(b))
    prob = build(16, 20, 23, [0.5, 0.5], b)
    st = solvers.init_state(prob)
    with pytest.raises(ValueError, match="sigma and mu_g must be positive"):
        solvers.sketch_step(st, prob, 0.0, 1.0)
    with pytest.raises(ValueError, match="unknown algorithm"):
        solvers.run(prob, "sketch-par", 1e-3, 1.0, 3)
    with pytest.raises(ValueError, match="theta_extrap"):
        solvers.run(prob, "sketch-seq", 1e-3, 1.0, 3, theta_extrap=-0.1)


def test_pdhg_matches_oracle():
    """pdhg_solve on the device (one imask_pdhg_step per iteration) against the
    float64 restatement of solvers.py:321-342, same operator norm."""
    side, na, nd, mu_g, mu = 32, 36, 47, 0.5, 0.5
    orc = ct_oracle.ProjectorOracle(side, na, nd)
    b = orc.apply(np.random.default_rng(12).random(side * side))
    k_norm = so.power_norm(orc.apply, orc.adjoint_apply, side * side)
    geom = ctmodel.Geometry(side, na, nd)
    K = ctmodel.projector_op(geom)
    fam = mrsketch.make_family(1, side, [1.0], mode="coarse")
    prob = solvers.make_problem(K, b, fam, proxlib.ridge_fn(mu_g), proxlib.quadratic_conjugate_fn(b),
                                coarse_projector=lambda f: ctmodel.coarse_projector(geom, f))
    x_ref = so.pdhg_solve(orc.apply, orc.adjoint_apply, b, mu_g, mu, 300, k_norm)
    x = solvers.pdhg_solve(prob, mu, iters=300, k_norm=k_norm)
    assert rel_l2(host(x), x_ref) <= 1e-4
    # the generic device path (a LinOp the engine does not recognise) agrees
    K_plain = linops.LinOp(K.domain_dim, K.range_dim, K.apply, K.adjoint_apply)
    prob2 = solvers.Problem(K=K_plain, b=prob.b, g=prob.g, f_conj=prob.f_conj, probs=prob.probs,
                            ops=prob.ops, fractions=prob.fractions, family=prob.family)
    x2 = solvers.pdhg_solve(prob2, mu, iters=300, k_norm=k_norm)
    assert rel_l2(host(x2), host(x)) <= 1e-5


def test_pdhg_reaches_dense_ridge_solution():
    """test_solvers.py:277-281 on the device: 5000 PDHG iterations reach the
    closed-form ridge solution (to float32 precision)."""
    side, na, nd = 16, 20, 23
    orc = ct_oracle.ProjectorOracle(side, na, nd)
    Kd = orc.to_csr().toarray()
    b = Kd @ np.random.default_rng(13).random(side * side)
    x_hat = np.linalg.solve(Kd.T @ Kd + np.eye(side * side), Kd.T @ b)
    prob = build(side, na, nd, [1.0], b, mu_g=1.0)
    x = solvers.pdhg_solve(prob, mu=1.0, iters=5000)
    assert rel_l2(host(x), x_hat) <= 2e-5


def test_run_pdhg_rows_and_ledger():
    side, na, nd = 32, 36, 47
    orc = ct_oracle.ProjectorOracle(side, na, nd)
    x_true = np.random.default_rng(14).random(side * side)
    b = orc.apply(x_true)
    prob = build(side, na, nd, [0.5, 0.5], b, mu_g=1e-2)
    rep = solvers.run(prob, "pdhg", 123.0, 1e-2, 20, record_every=5, x_ref=x_true)
    assert [r[0] for r in rep.rows] == [0, 5, 10, 15, 20]
    assert [r[1] for r in rep.rows] == [0.0, 10.0, 20.0, 30.0, 40.0]
    assert all(r[2] == 0 for r in rep.rows)
    x = solvers.pdhg_solve(prob, 1e-2, iters=20)
    assert np.array_equal(host(rep.x), host(x))
    rel = float(np.dot(host(x) - x_true, host(x) - x_true) / np.dot(x_true, x_true))
    assert abs(rep.rows[-1][3] - rel) <= 1e-6 * rel


@pytest.mark.parametrize("theta", [0.0, 0.7])
def test_sketch_seq_step_matches_oracle(theta):
    """ImaSk-Seq (solvers.py:265-305) on the device against its float64
    restatement: same level sequence, iterates and tables."""
    side, na, nd, probs = 64, 90, 91, [0.3, 0.3, 0.2, 0.2]
    orc = so.SketchedCT(side, na, nd, probs)
    b = orc.proj[1].apply(np.random.default_rng(15).random(side * side))
    prob = build(side, na, nd, probs, b)
    st = solvers.init_state(prob, seed=6)
    ost = so.init_state(orc, seed=6)
    for _ in range(10):
        solvers.sketch_seq_step(st, prob, 2e-4, 1e-2, theta)
        so.sketch_seq_step(ost, orc, b, 2e-4, 1e-2, 1e-2, theta)
        assert st.last_level == ost.last_level
    assert rel_l2(host(st.x), ost.x) <= 1e-4
    assert rel_l2(host(st.y), ost.y) <= 1e-4
    assert rel_l2(host(st.xbar), ost.xbar) <= 1e-4
    assert rel_l2(host(st.psi_sum), ost.psi_sum) <= 1e-4
    assert st.cost == ost.cost
    with pytest.raises(ValueError, match="theta_extrap"):
        solvers.sketch_seq_step(st, prob, 2e-4, 1e-2, 1.5)


def test_run_sketch_seq_and_saga_saddle():
    """run() for the sequential variant follows sketch_seq_step; saga-saddle with
    A_i = p_i K_i is the parallel sketched step (solvers.py:233-237)."""
    side, na, nd, probs = 32, 36, 47, [0.25] * 4
    orc = so.SketchedCT(side, na, nd, probs)
    b = orc.proj[1].apply(np.random.default_rng(16).random(side * side))
    prob = build(side, na, nd, probs, b)
    rep = solvers.run(prob, "sketch-seq", 1e-3, 1e-2, 12, record_every=4, seed=3,
                      theta_extrap=0.5)
    st = solvers.init_state(prob, seed=3)
    for _ in range(12):
        solvers.sketch_seq_step(st, prob, 1e-3, 1e-2, 0.5)
    assert np.array_equal(host(rep.x), host(st.x))
    assert [r[0] for r in rep.rows] == [0, 4, 8, 12]
    assert rep.rows[-1][1] == st.cost and rep.rows[-1][2] == st.last_level
    blocks = [linops.scale(op, float(p)) for op, p in zip(prob.ops, prob.probs)]
    assert solvers.verify_decomposition(prob.K, blocks, trials=1) <= solvers.DECOMPOSITION_TOL
    rep_s = solvers.run(prob, "saga-saddle", 1e-3, 1e-2, 12, record_every=4, seed=3)
    rep_p = solvers.run(prob, "sketch", 1e-3, 1e-2, 12, record_every=4, seed=3)
    assert np.array_equal(host(rep_s.x), host(rep_p.x))


def test_sharded_step_graph_with_nccl():
    """The multi-GPU step captured as one CUDA graph with its NCCL all-reduce
    (a real one-rank NCCL group on this GPU): replays are bit-identical to the
    eager sharded step and match the single-GPU step."""
    import json
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, os.path.join(repo, "tools", "sharded_graph_check.py")],
                         capture_output=True, text=True, timeout=600, cwd=repo)
    assert res.returncode == 0, res.stderr[-3000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["graph_eq_eager"], out
    assert out["rel_x_vs_single"] <= 1e-6 and out["rel_y_vs_single"] <= 1e-6, out
    assert out["graphs_captured"] >= 2, out


@pytest.mark.parametrize("args", [(1024, 1440, 1449, 6, 8), (256, 360, 363, 4, 12),
                                  (512, 720, 725, 5, 10, 2, 1)])
def test_fused_staging_bit_identical(args, monkeypatch):
    """x goes to the forward's value planes in one kernel (restriction or
    compensation fused into the pair-plane staging, k_stage32) or through
    restriction / compensation + k_prepare (IMASK_FUSED_STAGE=0): every level
    at both dual parities, then a seeded schedule; iterates bit-identical."""
    from paper_2412_10249_b200 import _lib
    from paper_2412_10249_b200 import dist as dist_mod

    side, na, nd, r, K = args[:5]
    world, rank = args[5:7] if len(args) > 5 else (1, 0)
    geom = ctmodel.Geometry(side, na, nd)
    b = np.random.default_rng(3).standard_normal(geom.m)
    fam = mrsketch.make_family(r, side, [1.0 / r] * r, mode="coarse")
    outs = {}
    try:
        for name, val in (("fused", None), ("two_kernels", "0")):
            if val is None:
                monkeypatch.delenv("IMASK_FUSED_STAGE", raising=False)
            else:
                monkeypatch.setenv("IMASK_FUSED_STAGE", val)
            _lib.check(_lib.lib().imask_reload_switches())
            ctmodel._plan_cache.clear()  # fresh plans take the switch
            prob = dist_mod.make_sharded_problem(geom, dist_mod.local_rows(geom, b, rank, world),
                                                 fam, 1e-2, rank, world)
            prob.engine.shard = solvers.Shard()  # the phases on one GPU, no collective
            st = solvers.init_state(prob, seed=4)
            gen = torch.Generator(device="cuda").manual_seed(0)
            st.x.copy_(torch.rand(side * side, device="cuda", generator=gen))
            prm = solvers._params(1e-6, 1e-2, 1e-2)
            levels = list(range(r)) * 2 + [int(v) for v in
                                           solvers.draw_levels(4, 0, K, prob.cum_probs)]
            for lv in levels:
                solvers._device_step(prob.engine, st, lv, prm)
            outs[name] = (host(st.x), host(st.y))
            del prob, st
    finally:
        monkeypatch.delenv("IMASK_FUSED_STAGE", raising=False)
        _lib.check(_lib.lib().imask_reload_switches())
        ctmodel._plan_cache.clear()
    assert np.array_equal(outs["fused"][0], outs["two_kernels"][0])
    assert np.array_equal(outs["fused"][1], outs["two_kernels"][1])


@pytest.mark.parametrize("side,na,nd,r,record_every", [(64, 90, 91, 3, 1), (64, 90, 91, 3, 4),
                                                       (48, 60, 69, 2, 1)])
def test_run_rows_match_an_explicit_step_loop(side, na, nd, r, record_every):
    """run()'s metric rows (device-side reductions, one read-back per run) and
    final iterate equal an explicit sketch_step loop recording the same
    iterations, also on a side the 32 x 32-tile kernels do not take (48)."""
    geom = ctmodel.Geometry(side, na, nd)
    probs = [1.0 / r] * r
    rng = np.random.default_rng(11)
    b = rng.random(geom.m)
    x_ref = rng.random(side * side).astype(np.float32)
    fam = mrsketch.make_family(r, side, probs, mode="coarse")
    K = ctmodel.projector_op(geom)
    pr = solvers.make_problem(K, b, fam, proxlib.ridge_fn(1e-2), proxlib.quadratic_conjugate_fn(b),
                              coarse_projector=lambda f: ctmodel.coarse_projector(geom, f))
    iters = 23
    rep = solvers.run(pr, "sketch", 2e-4, 1e-2, iters, record_every=record_every, seed=5,
                      x_ref=x_ref)
    # the same solve with every row from the stand-alone reduction
    st = solvers.init_state(pr, seed=5)
    rec = solvers._Recorder(torch.from_numpy(x_ref).cuda(), st.x.device, iters + 2, 0.0)
    rec.record(0, 0.0, 0, st.x)
    for k in range(1, iters + 1):
        solvers.sketch_step(st, pr, 2e-4, 1e-2)
        if k % record_every == 0 or k == iters:
            rec.record(k, st.cost, st.last_level, st.x)
    ref_rows = rec.rows()
    assert torch.equal(rep.x, st.x)
    assert len(rep.rows) == len(ref_rows)
    for a, c in zip(rep.rows, ref_rows):
        assert a[:3] == c[:3]
        assert abs(a[3] - c[3]) <= 1e-13 * abs(c[3])
        assert abs(a[4] - c[4]) <= 1e-9
    # seconds: non-decreasing device times
    secs = [row[5] for row in rep.rows]
    assert all(t1 >= t0 for t0, t1 in zip(secs, secs[1:]))


@pytest.mark.parametrize("side,na,nd,r", [(48, 60, 69, 2), (40, 45, 57, 3), (96, 120, 137, 6),
                                          (144, 100, 205, 5), (192, 180, 272, 7)])
def test_unusual_geometries_match_oracle(side, na, nd, r):
    """Geometries off the BASELINE grid (tools/geometry_sweep.py runs more): image
    sides the 32 x 32-tile kernels do not take run the any-size sketch and
    image-side kernels, whose tiles must still cover the whole image (a 48^2
    image once kept a 32^2 corner only); 96^2 with r = 6 has phi table rows of
    9, 36, ... values, which must still start 16-byte aligned for the 128-bit
    kernels (a misaligned-address fault once); 144^2 pairs the TMA forward with
    the any-size staging; r = 7 takes the 64-wide compensation tiles; 45 angles
    are not quad-closed. Compensation and 30 iterations against the float64
    oracle with non-uniform probabilities, and a second solve bit-identical."""
    probs = np.random.default_rng(side).dirichlet(np.ones(r) * 4.0)
    probs = [float(p) for p in probs / probs.sum()]
    geom = ctmodel.Geometry(side, na, nd)
    rng = np.random.default_rng(3)
    x0 = rng.random(side * side)
    fam = mrsketch.make_family(r, side, probs, mode="coarse")
    ops = so.SketchedCT(side, na, nd, probs)
    got = fam.apply_sketch(torch.from_numpy(x0.astype(np.float32)).cuda(), r).double().cpu().numpy()
    from oracle import sketch_oracle
    want = sketch_oracle.apply_sketch(x0.reshape(side, side), probs, r).ravel()
    assert rel_l2(got, want) <= 1e-5
    b = ops.proj[1].apply(x0) + 0.01 * rng.standard_normal(geom.m)
    K = ctmodel.projector_op(geom)
    pr = solvers.make_problem(K, b, fam, proxlib.ridge_fn(1e-2), proxlib.quadratic_conjugate_fn(b),
                              coarse_projector=lambda f: ctmodel.coarse_projector(geom, f))
    runs = []
    for _ in range(2):
        st = solvers.init_state(pr, seed=9)
        for _ in range(30):
            solvers.sketch_step(st, pr, 2e-4, 1e-2)
        runs.append((st.x.clone(), st.y.clone()))
    assert torch.equal(runs[0][0], runs[1][0]) and torch.equal(runs[0][1], runs[1][1])
    ost = so.init_state(ops, seed=9)
    for _ in range(30):
        so.sketch_step(ost, ops, b, 2e-4, 1e-2, 1e-2)
    assert rel_l2(runs[0][0].double().cpu().numpy(), ost.x) <= 1e-3
    assert rel_l2(runs[0][1].double().cpu().numpy(), ost.y) <= 1e-3

