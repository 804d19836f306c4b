"""Parity of the sketch-family kernels (3) with the reference (mrsketch.py)."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import solver_oracle, sketch_oracle
from paper_2412_10249_b200 import ctmodel, linops, mrsketch
from paper_2412_10249_b200.synth import ellipse_phantom

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.double().cpu().numpy()


def test_known_answers():
    # test_mrsketch.py:20-22, 33-38, known values
    assert host(mrsketch.decimate(dev([[1.0, 3.0], [5.0, 7.0]]), 2)).tolist() == [[4.0]]
    assert host(mrsketch.upsample(dev([[4.0]]), 2)).tolist() == [[4.0, 4.0], [4.0, 4.0]]
    assert np.array_equal(linops.densify(mrsketch.decimate_op(2, 2)), [[0.25, 0.25, 0.25, 0.25]])
    with pytest.raises(ValueError, match="divisible"):
        mrsketch.decimate(dev(np.zeros((6, 6))), 4)


def test_against_golden(g_sketch):
    x = g_sketch["x"]
    for f in (2, 4, 8):
        assert rel_l2(host(mrsketch.decimate(dev(x), f)), g_sketch[f"dec_f{f}"]) <= 1e-6
        up = mrsketch.upsample(mrsketch.decimate(dev(x), f), f)
        assert rel_l2(host(up), g_sketch[f"up_f{f}"]) <= 1e-6
    for name, probs in (("u3", [1 / 3] * 3), ("p4", [0.3, 0.3, 0.2, 0.2]), ("u6", [1 / 6] * 6)):
        fam = mrsketch.make_family(len(probs), 64, probs)
        for i in range(1, fam.r + 1):
            got = host(fam.apply_sketch(dev(x.ravel()), i))
            assert rel_l2(got, g_sketch[f"S_{name}_{i}"]) <= 1e-5, (name, i)


@pytest.mark.parametrize("side,r", [(1024, 6), (2048, 7), (16, 4), (8, 1)])
def test_unbiased_and_idempotent_full_size(side, r):
    """sum_i p_i S_i = I (test_mrsketch.py:121-138) and S_i^2 = S_i for i < r."""
    probs = [1.0 / r] * r
    fam = mrsketch.make_family(r, side, probs)
    x = dev(np.random.default_rng(side).standard_normal(side * side))
    assert float(torch.linalg.norm(fam.weighted_sum_apply(x) - x) / torch.linalg.norm(x)) <= 2e-6
    for i in range(1, r):
        once = fam.apply_sketch(x, i)
        twice = fam.apply_sketch(once, i)
        assert float(torch.linalg.norm(twice - once) / torch.linalg.norm(once)) <= 1e-6


def test_compensation_against_oracle_large():
    x = np.random.default_rng(9).standard_normal((512, 512))
    probs = [0.1, 0.2, 0.3, 0.15, 0.25]
    fam = mrsketch.make_family(5, 512, probs)
    got = host(fam.apply_sketch(dev(x.ravel()), 5))
    assert rel_l2(got, sketch_oracle.compensate(x, probs).ravel()) <= 1e-5


def test_scaled_adjoint_pairs():
    assert linops.adjoint_test(mrsketch.decimate_op(64, 4), trials=5, seed=0) <= 1e-6
    assert linops.adjoint_test(mrsketch.upsample_op(64, 8), trials=5, seed=1) <= 1e-6


def test_sketched_operators_vs_oracle():
    side, na, nd, probs = 64, 90, 91, [0.3, 0.3, 0.2, 0.2]
    geom = ctmodel.Geometry(side, na, nd)
    fam = mrsketch.make_family(4, side, probs, mode="coarse")
    K = ctmodel.projector_op(geom)
    ops = mrsketch.forward_family(fam, K, lambda f: ctmodel.coarse_projector(geom, f))
    orc = solver_oracle.SketchedCT(side, na, nd, probs)
    x = ellipse_phantom(side, 1).ravel()
    y = np.random.default_rng(4).standard_normal(geom.m)
    plan = ctmodel.get_plan(geom, 4, tuple(probs))
    for i0, op in enumerate(ops):
        assert op.meta is not None and op.meta.level == i0 + 1
        assert rel_l2(host(op.apply(dev(x))), orc.apply(i0, x)) <= 1e-4
        assert rel_l2(host(op.adjoint_apply(dev(y))), orc.adjoint_apply(i0, y)) <= 1e-4
        # the fused native entry points compute the same K_i / K_i^T
        assert rel_l2(host(plan.sketch_forward(i0 + 1, dev(x))), orc.apply(i0, x)) <= 1e-4
        assert rel_l2(host(plan.sketch_adjoint(i0 + 1, dev(y))), orc.adjoint_apply(i0, y)) <= 1e-4
