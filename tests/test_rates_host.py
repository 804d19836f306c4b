"""Step-size theory (rates.py:122-301) against the reference's outputs
(tests/golden/rates.npz from make_golden.py): scalar host arithmetic, no GPU."""

import numpy as np
import pytest

from conftest import golden
from paper_2412_10249_b200 import rates


@pytest.fixture(scope="module")
def g():
    return golden("rates.npz")


def _consts(row):
    L, Lb, Lbp, mp = (float(v) for v in row)
    return rates.RateConstants(L=L, Lbar=Lb, Lbar_p=Lbp, min_p=mp, mu_g=1.0, mu_fstar=1.0)


def test_plans_admissible_interval_and_theta(g):
    for idx, row in enumerate(g["cases"]):
        rc = _consts(row)
        c_bar = 1.0 / (1.0 + (rc.L * 1.01) ** 2 + (rc.Lbar_p * 1.01) ** 2)
        got = []
        for cf in (1e-3, 0.1, 0.5, 0.9):
            for rho in (0.05, 0.5, 0.95):
                pl = rates.plan_for(rc, cf * c_bar, rho)
                lo, hi = rates.admissible_interval(pl)
                got.append([pl.a, pl.b, pl.c, pl.c_bar, pl.rho, pl.alpha, pl.eta_star,
                            pl.sigma_star, pl.theta_star, lo, hi,
                            float(pl.theta_of(0.5 * pl.eta_star))])
        np.testing.assert_allclose(np.array(got), g[f"plans_{idx}"], rtol=1e-12, atol=0)


def test_optimal_step_grid_and_baseline(g):
    for idx, row in enumerate(g["cases"]):
        rc = _consts(row)
        best = rates.optimal_step(rc)
        free = rates.optimal_step(rc, rho=None, num_c=25, num_rho=20)
        got = np.array([[p.c, p.rho, p.eta_star, p.sigma_star, p.theta_star] for p in (best, free)])
        np.testing.assert_allclose(got, g[f"opt_{idx}"], rtol=1e-10)
        grid = rates.step_plan_grid(rc, num_c=7, num_rho=5)
        np.testing.assert_allclose(np.array([[p.c, p.rho, p.theta_star] for p in grid]),
                                   g[f"grid_{idx}"], rtol=1e-10)
        assert rates.sigma_baseline(rc.L, rc.Lbar) == pytest.approx(g[f"base_{idx}"][0], rel=1e-15)
        un = [rates.theta_unnormalized(s, mu, rc.L, rc.Lbar_p, rc.Lbar, rc.min_p, a, b)
              for s, mu, a, b in ((1e-3, 1.0, 2.0, 0.5), (0.2, 0.1, 0.7, 3.0))]
        np.testing.assert_allclose(un, g[f"unnorm_{idx}"], rtol=1e-13)


def test_argument_checks():
    rc = rates.RateConstants(L=2.0, Lbar=1.5, Lbar_p=3.0, min_p=0.25, mu_g=1.0, mu_fstar=1.0)
    with pytest.raises(ValueError, match="c must lie"):
        rates.plan_for(rc, 1.0, 0.5)
    with pytest.raises(ValueError, match="rho"):
        rates.plan_for(rc, 1e-4, 1.5)
    with pytest.raises(ValueError):
        rates.sigma_baseline(0.0, 1.0)
    with pytest.raises(ValueError):
        rates.theta_unnormalized(0.0, 1.0, 1.0, 1.0, 1.0, 0.5, 1.0, 1.0)
    phi, psi = rates.phi_psi(np.array([0.0, 0.1]), 0.1, 0.5, 2.0, 0.25)
    assert phi.shape == (2,) and psi[0] == pytest.approx(0.75)
