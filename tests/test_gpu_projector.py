"""Parity of the sm_100a projector kernels (1)/(2) with the reference operator.

Budget (north star): float32 projections and backprojections within 1e-4
relative L2 of the reference's float64 operator. Checks: the reference's
own matrices (golden), config A at every level, config D on sampled angles
(including the axis-parallel angles 0 and n/2 with integer detector offsets,
where the half-open tie rule decides), odd/even detector counts, the adjoint
identity, and size-independent properties at the full D / E sizes.
"""

import os

import numpy as np
import pytest
import torch
from scipy import sparse

from conftest import REPO, rel_l2
from oracle import ct_oracle, sketch_oracle
from paper_2412_10249_b200 import ctmodel, linops
from paper_2412_10249_b200.synth import CONFIGS, ellipse_phantom

pytestmark = pytest.mark.gpu
TOL = 1e-4  # north-star float32 budget (relative L2)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.double().cpu().numpy().ravel()


def test_golden_small_matrices(g_proj_small):
    rng = np.random.default_rng(0)
    idx = 0
    while f"c{idx}_meta" in g_proj_small:
        side, na, nd, f = (int(v) for v in g_proj_small[f"c{idx}_meta"])
        ref = sparse.csr_matrix(
            (g_proj_small[f"c{idx}_data"], g_proj_small[f"c{idx}_indices"],
             g_proj_small[f"c{idx}_indptr"]), shape=(na * nd, (side // f) ** 2))
        geom = ctmodel.Geometry(side, na, nd)
        op = ctmodel.coarse_projector(geom, f)
        x = rng.standard_normal(ref.shape[1])
        y = rng.standard_normal(ref.shape[0])
        assert rel_l2(host(op.apply(dev(x))), ref @ x) <= TOL, (side, na, nd, f)
        assert rel_l2(host(op.adjoint_apply(dev(y))), ref.T @ y) <= TOL, (side, na, nd, f)
        # densified columns: every matrix entry within float32 rounding
        if ref.shape[1] <= 256:
            dense = linops.densify(op)
            assert np.max(np.abs(dense - ref.toarray())) <= 1e-5 * max(1, f), (side, na, nd, f)
        idx += 1


def test_single_pixel_centre_chord():
    # test_ctmodel.py:39-42: a ray through the centre of a unit pixel has chord 1
    geom = ctmodel.Geometry(1, 1, 1)
    assert host(ctmodel.project(geom, dev([1.0])))[0] == 1.0


def test_config_A_every_level(g_proj_A):
    cfg = CONFIGS["A"]
    geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    x, y = g_proj_A["x"], g_proj_A["y"]
    for f in (1, 2, 4):
        op = ctmodel.coarse_projector(geom, f)
        xl = sketch_oracle.decimate(x, f).ravel()
        assert rel_l2(host(op.apply(dev(xl))), g_proj_A[f"fwd_f{f}"]) <= TOL
        assert rel_l2(host(op.adjoint_apply(dev(y))), g_proj_A[f"adj_f{f}"]) <= TOL


def test_config_A_axis_rows_exact(g_proj_A):
    """Rows theta = 0 and pi/2 (every ray on a gridline) carry the tie rule."""
    cfg = CONFIGS["A"]
    geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    x = g_proj_A["x"]
    for f in (1, 2, 4):
        got = host(ctmodel.coarse_projector(geom, f).apply(
            dev(sketch_oracle.decimate(x, f).ravel()))).reshape(cfg.n_angles, cfg.n_det)
        ref = g_proj_A[f"fwd_f{f}"].reshape(cfg.n_angles, cfg.n_det)
        for a in (0, cfg.n_angles // 2):
            assert rel_l2(got[a], ref[a]) <= 1e-6, (f, a)


def test_config_D_sampled_angles(g_proj_D):
    cfg = CONFIGS["D"]
    geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    sel = g_proj_D["angles"]
    x = ellipse_phantom(cfg.side, 0)
    yfull = np.zeros((cfg.n_angles, cfg.n_det))
    yfull[sel] = g_proj_D["y"].reshape(len(sel), cfg.n_det)
    for f in (1, 2, 4, 8, 16, 32):  # every level of config D
        op = ctmodel.coarse_projector(geom, f)
        sino = host(op.apply(dev(sketch_oracle.decimate(x, f).ravel()))).reshape(cfg.n_angles, -1)
        ref = g_proj_D[f"fwd_f{f}"].reshape(len(sel), cfg.n_det)
        assert rel_l2(sino[sel], ref) <= TOL
        for k in range(len(sel)):
            assert rel_l2(sino[sel[k]], ref[k]) <= TOL, (f, sel[k])
        bp = host(op.adjoint_apply(dev(yfull)))
        if f == 1:
            assert rel_l2(bp[g_proj_D["pix"]], g_proj_D["adj_f1_at_pix"]) <= TOL
        elif f"pix_f{f}" in g_proj_D:
            assert rel_l2(bp[g_proj_D[f"pix_f{f}"]], g_proj_D[f"adj_f{f}"]) <= TOL, f
        else:
            assert rel_l2(bp, g_proj_D[f"adj_f{f}"]) <= TOL, f


@pytest.mark.parametrize("side,na,nd,factors", [
    (256, 360, 363, (1, 2, 4, 8)),   # config B
    (48, 30, 70, (1, 2, 3, 4, 6)),   # even detector count, non-power-of-two factors
    (40, 17, None, (1, 5)),          # odd angle count (no pi/2 angle)
])
def test_against_oracle_live(side, na, nd, factors):
    geom = ctmodel.Geometry(side, na, nd)
    rng = np.random.default_rng(side)
    for f in factors:
        orc = ct_oracle.ProjectorOracle(side, na, geom.n_detectors, f)
        op = ctmodel.coarse_projector(geom, f)
        x = rng.random(orc.domain_dim)
        y = rng.standard_normal(orc.range_dim)
        assert rel_l2(host(op.apply(dev(x))), orc.apply(x)) <= TOL, f
        assert rel_l2(host(op.adjoint_apply(dev(y))), orc.adjoint_apply(y)) <= TOL, f


def test_config_C_sampled_rows():
    cfg = CONFIGS["C"]
    geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    sel = np.array([0, 1, 179, 180, 181, 359, 360, 361, 540, 719])
    x = ellipse_phantom(cfg.side, 2)
    for f in (1, 4, 16):
        xl = sketch_oracle.decimate(x, f).ravel()
        got = host(ctmodel.coarse_projector(geom, f).apply(dev(xl))).reshape(cfg.n_angles, -1)
        orc = ct_oracle.ProjectorOracle(cfg.side, cfg.n_angles, cfg.n_det, f, angle_idx=sel)
        assert rel_l2(got[sel].ravel(), orc.apply(xl)) <= TOL, f


@pytest.mark.parametrize("key", ["A", "B", "D"])
def test_adjoint_identity_every_level(key):
    cfg = CONFIGS[key]
    geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    for lev in range(cfg.levels):
        f = 2 ** lev
        gap = linops.adjoint_test(ctmodel.coarse_projector(geom, f), trials=3, seed=f)
        assert gap <= 2e-6, (key, f, gap)


@pytest.mark.parametrize("key", ["D", "E"])
def test_full_size_properties(key):
    """At the BASELINE's full sizes: linearity, theta=0 mass conservation, coarse == replicated."""
    cfg = CONFIGS[key]
    geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    x = ellipse_phantom(cfg.side, 1).ravel()
    rng = np.random.default_rng(1)
    z = rng.standard_normal(cfg.side * cfg.side)
    K = ctmodel.projector_op(geom)
    kx, kz = K.apply(dev(x)), K.apply(dev(z))
    lin = K.apply(dev(2.0 * x - 3.0 * z))
    assert float(torch.linalg.norm(lin - (2 * kx - 3 * kz)) / torch.linalg.norm(lin)) <= 1e-5
    sino = host(kx).reshape(cfg.n_angles, cfg.n_det)
    # theta = 0: every pixel lands whole in exactly one bin (test_ctmodel.py:56-60)
    assert abs(sino[0].sum() - x.sum()) <= 1e-5 * x.sum()
    assert abs(sino[cfg.n_angles // 2].sum() - x.sum()) <= 1e-5 * x.sum()
    for f in (2, 8, 2 ** (cfg.levels - 1)):
        xl = sketch_oracle.decimate(x.reshape(cfg.side, cfg.side), f)
        via_coarse = host(ctmodel.coarse_projector(geom, f).apply(dev(xl.ravel())))
        via_full = host(K.apply(dev(sketch_oracle.upsample(xl, f).ravel())))
        assert rel_l2(via_coarse, via_full) <= TOL, f


def test_projections_repeat_bit_for_bit():
    """Every launch of a projector gives the same bits (config D, every kernel
    family: TMA one- and two-detector forwards, the L1 quad forward, pair /
    unrolled / bin-loop adjoints with their split planes): a shared-memory or
    barrier race would show as run-to-run differences, which compute-sanitizer
    (closed on the pool) cannot be asked about."""
    cfg = CONFIGS["D"]
    geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    plan = ctmodel.get_plan(geom)
    gen = torch.Generator(device="cuda").manual_seed(5)
    y = torch.randn(geom.m, device="cuda", generator=gen)
    for f in (1, 2, 4, 8, 32):
        u = torch.rand((cfg.side // f) ** 2, device="cuda", generator=gen)
        s0, b0 = plan.project(u, f).clone(), plan.backproject(y, f).clone()
        for _ in range(5):
            # other work in between changes the CTA schedule from launch to launch
            plan.backproject(y, 2 * f if f < 32 else 1)
            assert torch.equal(plan.project(u, f), s0), f
            assert torch.equal(plan.backproject(y, f), b0), f


def test_empty_and_degenerate_inputs():
    geom = ctmodel.Geometry(16, 20, 23)
    K = ctmodel.projector_op(geom)
    assert torch.count_nonzero(K.apply(torch.zeros(256, device="cuda"))) == 0
    assert torch.count_nonzero(K.adjoint_apply(torch.zeros(geom.m, device="cuda"))) == 0
    with pytest.raises(linops.DimensionMismatch, match="domain dim 256"):
        linops.apply(K, np.zeros(255))
    with pytest.raises(linops.DimensionMismatch, match="range dim 460"):
        linops.adjoint(K, np.zeros(10))
    with pytest.raises(ValueError, match="not divisible by factor 3"):
        ctmodel.coarse_projector(geom, 3)
    # an empty angle slab projects to an empty sinogram and backprojects to zero
    plan = ctmodel.Plan(geom, angle_begin=5, angle_end=5)
    out = plan.project(torch.ones(256, device="cuda"), 1)
    assert out.numel() == 0
    bp = plan.backproject(torch.zeros(0, device="cuda"), 1)
    assert torch.count_nonzero(bp) == 0


def test_slab_rows_match_full():
    geom = ctmodel.Geometry(64, 90, 91)
    x = dev(sketch_oracle.decimate(ellipse_phantom(64, 5), 2).ravel())
    y = np.random.default_rng(2).standard_normal(geom.m)
    full = host(ctmodel.get_plan(geom).project(x, 2)).reshape(90, 91)
    bp_sum = np.zeros(32 * 32)
    for rank in range(3):
        b, e = ctmodel.slab_bounds(90, rank, 3)
        plan = ctmodel.Plan(geom, angle_begin=b, angle_end=e)
        part = host(plan.project(x, 2)).reshape(e - b, 91)
        # the full plan traces mirror pairs (a, n-a) from angle a's parameters, the slab
        # plans trace each angle from its own: equal up to float32 rounding
        assert rel_l2(part, full[b:e]) <= 1e-6
        bp_sum += host(plan.backproject(dev(y.reshape(90, 91)[b:e]), 2))
    ref = host(ctmodel.get_plan(geom).backproject(dev(y), 2))
    assert rel_l2(bp_sum, ref) <= 1e-6


@pytest.mark.parametrize("n_angles,world", [(90, 2), (90, 3), (91, 4), (180, 8), (360, 2)])
def test_mirror_closed_shards_match_full(n_angles, world):
    """Every shard of shard_angles runs the symmetric kernels; its rows equal the
    full plan's rows, and the shards' backprojections sum to the full one.
    (360 angles on 2 ranks: the block-cyclic quad shards.)"""
    if n_angles == 360:
        a0 = ctmodel.shard_angles(n_angles, 0, world)
        assert 6 in a0 and 7 not in a0 and 15 in a0  # groups of 8 forward entries alternate
    geom = ctmodel.Geometry(64, n_angles, 91)
    x = dev(ellipse_phantom(64, 6).ravel())
    y = np.random.default_rng(3).standard_normal(geom.m).reshape(n_angles, 91)
    full_plan = ctmodel.get_plan(geom)
    assert full_plan.symmetric
    for f in (1, 4):
        u = x if f == 1 else dev(sketch_oracle.decimate(ellipse_phantom(64, 6), f).ravel())
        full = host(full_plan.project(u, f)).reshape(n_angles, 91)
        ref = host(full_plan.backproject(dev(y), f))
        bp_sum = np.zeros((64 // f) ** 2)
        for rank in range(world):
            idx = list(ctmodel.shard_angles(n_angles, rank, world))
            plan = ctmodel.Plan(geom, angles=idx)
            assert plan.symmetric
            assert plan.quad_forward == (n_angles % 4 == 0)
            part = host(plan.project(u, f)).reshape(len(idx), 91)
            assert rel_l2(part, full[idx]) <= 1e-6
            bp_sum += host(plan.backproject(dev(y[idx]), f))
        assert rel_l2(bp_sum, ref) <= 1e-6


@pytest.mark.parametrize("geom_args", [(1024, 1440, 1449, 1), (1024, 1440, 1449, 2),
                                       (1024, 1440, 1449, 8), (256, 360, 363, 1),
                                       (256, 360, 363, 2), (256, 360, 363, 4)])
def test_forward_paths_bit_identical(geom_args, monkeypatch):
    """The four-ray (quad) TMA forward, the pair TMA forward and the L1 forward
    trace the same rays with the same arithmetic: bit-identical sinograms, with
    the difference pairs read from the difference planes or formed from the
    value planes (P[c+1] - P[c]), and with one or two detectors per thread.
    The path switches are environment variables re-read by
    imask_reload_switches; each variant gets a fresh plan."""
    from paper_2412_10249_b200 import _lib

    side, na, nd, f = geom_args
    geom = ctmodel.Geometry(side, na, nd)
    n = side // f
    gen = torch.Generator(device="cuda").manual_seed(0)
    u = torch.rand(n * n, device="cuda", generator=gen)
    outs = {}
    variants = (("quad", {}), ("pair", {"IMASK_NO_QUAD": "1"}), ("l1", {"IMASK_NO_TMA": "1"}),
                ("quad_planes", {"IMASK_FWD_VAL": "0"}),
                ("pair_planes", {"IMASK_NO_QUAD": "1", "IMASK_FWD_VAL": "0"}),
                ("l1_planes", {"IMASK_NO_TMA": "1", "IMASK_FWD_VAL_L1": "0"}),
                # one detector per thread (f >= 2 default: two)
                ("one_det", {"IMASK_FWD_TWO_DET": "0"}),
                ("one_det_planes", {"IMASK_FWD_TWO_DET": "0", "IMASK_FWD_VAL": "0"}),
                ("pair_one_det", {"IMASK_NO_QUAD": "1", "IMASK_FWD_TWO_DET": "0"}))
    names = {k for _, env in variants for k in env}
    try:
        for name, env in variants:
            for k in names:
                monkeypatch.delenv(k, raising=False)
            for k, v in env.items():
                monkeypatch.setenv(k, v)
            _lib.check(_lib.lib().imask_reload_switches())
            plan = ctmodel.Plan(geom)
            outs[name] = host(plan.project(u, f))
            del plan
    finally:
        for k in names:
            monkeypatch.delenv(k, raising=False)
        _lib.check(_lib.lib().imask_reload_switches())
    for name in outs:
        assert np.array_equal(outs["quad"], outs[name]), name

@pytest.mark.parametrize("geom_args,world,rank", [((1024, 1440, 1449), 1, 0), ((256, 360, 363), 1, 0),
                                                  ((256, 360, 363), 4, 1), ((64, 90, 91), 1, 0)])
def test_adjoint_row_pairs_bit_identical(geom_args, world, rank, monkeypatch):
    """The f=1 symmetric adjoint on row pairs (single-bin windows shared by two
    vertically adjacent pixels; an A/B variant, off by default) and the
    pair-window kernel evaluate the same weights and sums in the same order:
    bit-identical backprojections."""
    from paper_2412_10249_b200 import _lib

    geom = ctmodel.Geometry(*geom_args)
    rows = ctmodel.shard_angles(geom.n_angles, rank, world)
    gen = torch.Generator(device="cuda").manual_seed(1)
    y = torch.randn(len(rows) * geom.n_detectors, device="cuda", generator=gen)
    outs = {}
    try:
        for name, val in (("rows", "1"), ("pairs", "0")):
            monkeypatch.setenv("IMASK_ADJ_ROW_PAIR", val)
            _lib.check(_lib.lib().imask_reload_switches())
            plan = ctmodel.Plan(geom, angles=rows)
            assert plan.symmetric
            outs[name] = host(plan.backproject(y, 1))
            del plan
    finally:
        monkeypatch.delenv("IMASK_ADJ_ROW_PAIR", raising=False)
        _lib.check(_lib.lib().imask_reload_switches())
    assert np.array_equal(outs["rows"], outs["pairs"])
