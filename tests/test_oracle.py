"""Pin the CPU oracle against the reference's own outputs (tests/golden/, made by
tests/golden/make_golden.py from /root/reference). CPU only."""

import os

import numpy as np
import pytest
from scipy import sparse

from conftest import REFERENCE_SRC, rel_l2
from oracle import ct_oracle, sketch_oracle, solver_oracle
from paper_2412_10249_b200.synth import CONFIGS, add_gaussian_noise, ellipse_phantom


def test_ray_matrix_small_geometries(g_proj_small):
    idx = 0
    while f"c{idx}_meta" in g_proj_small:
        side, na, nd, f = (int(v) for v in g_proj_small[f"c{idx}_meta"])
        ref = sparse.csr_matrix(
            (g_proj_small[f"c{idx}_data"], g_proj_small[f"c{idx}_indices"],
             g_proj_small[f"c{idx}_indptr"]),
            shape=(na * nd, (side // f) ** 2),
        )
        mine = ct_oracle.ProjectorOracle(side, na, nd, f).to_csr()
        assert abs(mine - ref).max() <= 1e-12, (side, na, nd, f)
        assert mine.nnz == ref.nnz, (side, na, nd, f)
        idx += 1
    assert idx >= 8


def test_config_A_every_level(g_proj_A):
    cfg = CONFIGS["A"]
    x = g_proj_A["x"]
    assert np.array_equal(x, ellipse_phantom(cfg.side, 0))
    for f in (1, 2, 4):
        op = ct_oracle.ProjectorOracle(cfg.side, cfg.n_angles, cfg.n_det, f)
        xl = sketch_oracle.decimate(x, f).ravel()
        assert rel_l2(op.apply(xl), g_proj_A[f"fwd_f{f}"]) <= 1e-13
        assert rel_l2(op.adjoint_apply(g_proj_A["y"]), g_proj_A[f"adj_f{f}"]) <= 1e-13


def test_config_D_sampled_angles(g_proj_D):
    cfg = CONFIGS["D"]
    x = ellipse_phantom(cfg.side, 0)
    sel = g_proj_D["angles"]
    for f in (1, 32):
        op = ct_oracle.ProjectorOracle(cfg.side, cfg.n_angles, cfg.n_det, f, angle_idx=sel)
        assert rel_l2(op.apply(sketch_oracle.decimate(x, f).ravel()), g_proj_D[f"fwd_f{f}"]) <= 1e-11
        bp = op.adjoint_apply(g_proj_D["y"])
        if f == 1:
            assert rel_l2(bp[g_proj_D["pix"]], g_proj_D["adj_f1_at_pix"]) <= 1e-11
        else:
            assert rel_l2(bp, g_proj_D["adj_f32"]) <= 1e-11


def test_tie_rule_axis_angles():
    # theta = 0 with an odd detector count: every ray lies on a gridline and belongs to the
    # pixel column on its right (ctmodel.py:99-114); the mass of column j+N/2 lands in bin j.
    side, nd = 8, 11
    op = ct_oracle.ProjectorOracle(side, 2, nd, 1)
    img = np.zeros((side, side))
    img[:, 5] = 1.0  # column 5 spans x in [1, 2): only the ray t = 1 claims it
    sino = op.apply(img.ravel()).reshape(2, nd)
    t = ct_oracle.offsets(nd)
    assert sino[0, np.nonzero(t == 1.0)[0][0]] == side
    assert sino[0].sum() == side
    # theta = pi/2: rays run along x at y = t; row 5 spans y in [1, 2)
    img = np.zeros((side, side))
    img[5, :] = 1.0
    sino = op.apply(img.ravel()).reshape(2, nd)
    assert sino[1, np.nonzero(t == 1.0)[0][0]] == side


def test_sketch_family(g_sketch):
    x = g_sketch["x"]
    for f in (2, 4, 8):
        assert np.allclose(sketch_oracle.decimate(x, f), g_sketch[f"dec_f{f}"], rtol=0, atol=1e-14)
        assert np.allclose(
            sketch_oracle.upsample(sketch_oracle.decimate(x, f), f), g_sketch[f"up_f{f}"],
            rtol=0, atol=1e-14,
        )
    for name, probs in (("u3", [1 / 3] * 3), ("p4", [0.3, 0.3, 0.2, 0.2]), ("u6", [1 / 6] * 6)):
        for i in range(1, len(probs) + 1):
            got = sketch_oracle.apply_sketch(x, probs, i).ravel()
            assert np.max(np.abs(got - g_sketch[f"S_{name}_{i}"])) <= 1e-12


def test_level_rng_bit_exact(g_rng):
    seeds = [int(s) for s in g_rng["seeds"]]
    for pname, p in (("u3", [1 / 3] * 3), ("u6", [1 / 6] * 6), ("p4", [0.3, 0.3, 0.2, 0.2]),
                     ("u7", [1 / 7] * 7)):
        for si, seed in enumerate(seeds):
            got = solver_oracle.level_schedule(seed, 0, 5000, p)
            assert np.array_equal(got, g_rng[f"levels_{pname}_s{si}"].astype(np.int64))
    u = [solver_oracle.uniform_at(12345, k) for k in range(256)]
    assert np.array_equal(np.array(u), g_rng["uniform_s12345"])


def test_solver_trajectory_A(g_solver_A):
    cfg = CONFIGS["A"]
    x_true = ellipse_phantom(cfg.side, 0)
    ops = solver_oracle.SketchedCT(cfg.side, cfg.n_angles, cfg.n_det, [1.0 / 3] * 3)
    sino = ops.proj[1].apply(x_true.ravel())
    b = add_gaussian_noise(sino, cfg.kappa, 1)
    assert rel_l2(b, g_solver_A["b"]) <= 1e-13
    st = solver_oracle.init_state(ops, seed=int(g_solver_A["seed"]))
    sigma, mu = float(g_solver_A["sigma"]), float(g_solver_A["mu"])
    for k in range(1, 201):
        solver_oracle.sketch_step(st, ops, g_solver_A["b"], sigma, mu, cfg.mu_g)
        if k in (18, 200):
            assert rel_l2(st.x, g_solver_A[f"x_{k}"]) <= 1e-11
            assert rel_l2(st.y, g_solver_A[f"y_{k}"]) <= 1e-11
            assert st.cost == float(g_solver_A[f"cost_{k}"])
    assert np.array_equal(np.array(st.levels) + 1, g_solver_A["levels"].astype(np.int64))


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference tree not present")
def test_against_live_reference_odd_and_even_detectors():
    import sys

    sys.path.insert(0, REFERENCE_SRC)
    from mrtomo import ctmodel

    for side, na, nd, f in ((24, 12, 35, 1), (24, 12, 34, 2), (48, 30, None, 4)):
        g = ctmodel.Geometry(side, na, nd)
        ref = ctmodel.ray_matrix(side // f, float(f), g.angles, g.offsets)
        mine = ct_oracle.ProjectorOracle(side, na, g.n_detectors, f).to_csr()
        assert abs(mine - ref).max() <= 1e-12


def test_tv_oracle_pinned_to_reference(g_tv):
    """oracle/prox_oracle.py reproduces the reference's prox_tv_nonneg
    (proxlib.py:102-148) on the golden inputs."""
    from oracle import prox_oracle as po

    for side in (16, 40, 64):
        sigma, mu_g = g_tv[f"par_{side}"]
        out = po.prox_tv_nonneg(g_tv[f"xp_{side}"], sigma, mu_g)
        assert np.max(np.abs(out - g_tv[f"out_{side}"])) <= 1e-12
    out = po.prox_tv_nonneg(g_tv["xp_step"], 0.8, 0.5, inner_iters=4000, inner_tol=1e-13)
    assert np.max(np.abs(out - g_tv["out_step"])) <= 1e-12


@pytest.mark.parametrize("name,min_f", [("C", 2), ("E", 16)])
def test_sampled_angles_large_configs(name, min_f):
    """The oracle against the reference's ray_matrix rows at configs C and E
    (coarse levels: the fine ones take minutes on one core)."""
    from conftest import golden

    cfg = CONFIGS[name]
    g = golden(f"proj_{name}_sampled.npz")
    sel = g["angles"].astype(np.int64)
    x = ellipse_phantom(cfg.side, 0)
    y = g["y"].astype(np.float64)
    for lv in range(cfg.levels):
        f = 2 ** lv
        if f < min_f:
            continue
        op = ct_oracle.ProjectorOracle(cfg.side, cfg.n_angles, cfg.n_det, f, sel)
        xl = sketch_oracle.decimate(x, f).ravel()
        assert rel_l2(op.apply(xl), g[f"fwd_f{f}"]) <= 1e-12, (name, f)
        bp = op.adjoint_apply(y)
        if f"pix_f{f}" in g:
            bp = bp[g[f"pix_f{f}"]]
        assert rel_l2(bp, g[f"adj_f{f}"]) <= 1e-12, (name, f)


def test_solver_trajectory_C_first_steps():
    """The oracle's sketch_step against the reference trajectory at config C
    (golden solver_C.npz), through the first 26 iterations."""
    from conftest import golden

    g = golden("solver_C.npz")
    cfg = CONFIGS["C"]
    orc = solver_oracle.SketchedCT(cfg.side, cfg.n_angles, cfg.n_det, [1.0 / cfg.levels] * cfg.levels,
                                   csr=False)
    b = g["b"].astype(np.float64)
    st = solver_oracle.init_state(orc, seed=int(g["seed"]))
    for _ in range(26):
        solver_oracle.sketch_step(st, orc, b, float(g["sigma"]), float(g["mu"]), cfg.mu_g)
    assert [lv + 1 for lv in st.levels] == g["levels"][:26].astype(int).tolist()
    assert rel_l2(st.x, g["x_26"]) <= 1e-6 and rel_l2(st.y, g["y_26"]) <= 1e-6
