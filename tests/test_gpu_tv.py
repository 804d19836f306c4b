"""TV + nonnegativity prox on the device against the
reference's own outputs (golden) and the float64 oracle; the reference test
cases of test_proxlib.py:101-145 on the device."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import prox_oracle as po
from paper_2412_10249_b200 import linops, proxlib

pytestmark = pytest.mark.gpu


def host(t):
    torch.cuda.synchronize()
    return t.double().cpu().numpy().ravel()


def test_matches_reference_golden(g_tv):
    for side in (16, 40, 64):
        sigma, mu_g = g_tv[f"par_{side}"]
        out = host(proxlib.prox_tv_nonneg(g_tv[f"xp_{side}"], sigma, mu_g))
        assert np.max(np.abs(out - g_tv[f"out_{side}"])) <= 2e-5, side
    out = host(proxlib.prox_tv_nonneg(g_tv["xp_step"], 0.8, 0.5, inner_iters=4000,
                                      inner_tol=1e-13))
    assert np.max(np.abs(out - g_tv["out_step"])) <= 1e-5


@pytest.mark.parametrize("side", [32, 100, 256])
def test_matches_oracle(side):
    xp = np.random.default_rng(side).standard_normal(side * side)
    out = host(proxlib.prox_tv_nonneg(xp, 0.7, 0.4))
    ref = po.prox_tv_nonneg(xp, 0.7, 0.4)
    assert rel_l2(out, ref) <= 1e-5


def test_reference_properties():
    x = np.full(64, 0.8)
    assert np.max(np.abs(host(proxlib.prox_tv_nonneg(x, 0.5, 1.0)) - x)) <= 1e-6
    assert np.all(host(proxlib.prox_tv_nonneg(np.full(64, -1.0), 0.5, 1.0)) == 0.0)
    out = host(proxlib.prox_tv_nonneg(np.random.default_rng(0).standard_normal(256), 1.0, 0.5))
    assert out.min() >= 0.0
    with pytest.raises(ValueError):
        proxlib.prox_tv_nonneg(x, 0.0, 1.0)
    with pytest.raises(ValueError, match="square"):
        proxlib.prox_tv_nonneg(np.ones(10), 1.0, 1.0)


def test_gradient_op_and_value():
    op = proxlib.gradient_op(8)
    assert linops.adjoint_test(op, trials=10, seed=0) <= 1e-5
    res = linops.power_method(proxlib.gradient_op(16), tol=1e-7, max_iter=5000, seed=1)
    assert res.norm <= np.sqrt(proxlib.GRAD_NORM_SQ) + 1e-3
    x = np.random.default_rng(3).random(64)
    g = po.grad(x, 8)
    assert proxlib.tv_value(x, 8, 0.5) == pytest.approx(0.5 * np.sum(np.hypot(g[:64], g[64:])),
                                                        rel=1e-6)
    fn = proxlib.tv_nonneg_fn(0.5)
    assert fn.kind == "tv_nonneg" and fn.strong_convexity == 0.0
    assert fn.value(-x) == float("inf")


def test_early_stop_on_converged_problem():
    """The relative-progress stop (device flag) leaves a constant image exactly."""
    x = np.full(32 * 32, 0.25)
    out = host(proxlib.prox_tv_nonneg(x, 1.0, 1.0, inner_iters=500, inner_tol=1e-6))
    assert np.max(np.abs(out - 0.25)) <= 1e-7


def test_imask_step_with_tv_regulariser():
    """ImaSk with g = TV + nonnegativity (the paper's section 4.5 setting): the
    native step runs the TV prox after the image-side update, inside the step
    graph; iterates match the float64 oracle step with the oracle TV prox."""
    from oracle import solver_oracle as so
    from paper_2412_10249_b200 import ctmodel, mrsketch, solvers

    side, na, nd, probs, mu_tv = 64, 90, 91, [0.3, 0.3, 0.2, 0.2], 2e-3
    orc = so.SketchedCT(side, na, nd, probs)
    b = orc.proj[1].apply(np.random.default_rng(17).random(side * side))
    geom = ctmodel.Geometry(side, na, nd)
    fam = mrsketch.make_family(len(probs), side, probs, mode="coarse")
    prob = solvers.make_problem(ctmodel.projector_op(geom), b, fam, proxlib.tv_nonneg_fn(mu_tv),
                                proxlib.quadratic_conjugate_fn(b),
                                coarse_projector=lambda f: ctmodel.coarse_projector(geom, f))
    assert prob.engine is not None
    st = solvers.init_state(prob, seed=2)
    ost = so.init_state(orc, seed=2)
    gprox = lambda p, s: po.prox_tv_nonneg(p, s, mu_tv)
    for _ in range(8):
        solvers.sketch_step(st, prob, 2e-4, 1e-2)
        so.sketch_step(ost, orc, b, 2e-4, 1e-2, 0.0, gprox=gprox)
    assert st.last_level == ost.last_level
    assert rel_l2(host(st.x), ost.x) <= 1e-4
    assert host(st.x).min() >= 0.0
    # the graph path (run) gives the same iterates as the eager steps
    rep = solvers.run(prob, "sketch", 2e-4, 1e-2, 8, record_every=8, seed=2)
    assert rel_l2(host(rep.x), host(st.x)) <= 1e-6
