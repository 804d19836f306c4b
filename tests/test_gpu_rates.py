"""Rate constants on the device against dense float64
linear algebra, as test_rates.py:26-94 checks the reference."""

import numpy as np
import pytest

from oracle import ct_oracle, sketch_oracle
from paper_2412_10249_b200 import ctmodel, linops, mrsketch, rates

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K16():
    return ctmodel.projector_op(ctmodel.Geometry(16, 20, 23))


@pytest.fixture(scope="module")
def dense_blocks():
    """0.25 * K S_i, i = 1..4, in float64 from the oracle (exact sketch ops)."""
    Kd = ct_oracle.ProjectorOracle(16, 20, 23).to_csr().toarray()
    eye = np.eye(256)
    out = []
    for i in (1, 2, 3, 4):
        S = np.stack([sketch_oracle.apply_sketch(eye[:, j].reshape(16, 16), [0.25] * 4, i).ravel()
                      for j in range(256)], axis=1)
        out.append(0.25 * Kd @ S)
    return out


def test_ct_family_matches_dense_stacked_svd(K16, dense_blocks):
    fam = mrsketch.make_family(4, 16, [0.25] * 4)
    c = rates.estimate_constants(fam, K16, mu_g=1.0, mu_fstar=1.0, tol=1e-7, max_iter=5000)
    L_exact = np.linalg.svd(sum(dense_blocks), compute_uv=False)[0]
    exact = {}
    for name, w in (("Lbar", 1.0), ("Lbar_p", 4.0)):
        primal = np.linalg.eigvalsh(sum(w * A.T @ A for A in dense_blocks))[-1]
        dual = np.linalg.eigvalsh(sum(w * A @ A.T for A in dense_blocks))[-1]
        exact[name] = np.sqrt(max(primal, dual))
    assert c.L == pytest.approx(L_exact, rel=1e-4)
    assert c.Lbar == pytest.approx(exact["Lbar"], rel=1e-4)
    assert c.Lbar_p == pytest.approx(exact["Lbar_p"], rel=1e-4)
    assert c.Lbar <= c.Lbar_p * (1 + 1e-6)


def test_single_level_all_equal(K16):
    c = rates.estimate_constants(mrsketch.make_family(1, 16, [1.0]), K16, 1.0, 1.0, tol=1e-7,
                                 max_iter=5000)
    assert c.L == pytest.approx(c.Lbar, rel=1e-4)
    assert c.L == pytest.approx(c.Lbar_p, rel=1e-4)


def test_identical_blocks_remark():
    n = 4
    a = np.random.default_rng(0).standard_normal((6, 5))
    nc = np.linalg.svd(a, compute_uv=False)[0]
    L, Lbar, Lbar_p, conv = rates.estimate_block_norms([linops.from_matrix(a)] * n,
                                                       np.full(n, 1.0 / n), tol=1e-7,
                                                       max_iter=5000)
    assert L == pytest.approx(n * nc, rel=1e-4)
    assert Lbar == pytest.approx(np.sqrt(n) * nc, rel=1e-4)
    assert Lbar_p == pytest.approx(n * nc, rel=1e-4)


def test_normalization_scaling(K16):
    fam = mrsketch.make_family(2, 16, [0.5, 0.5])
    a = rates.estimate_constants(fam, K16, 1.0, 1.0, tol=1e-7, max_iter=3000)
    b = rates.estimate_constants(fam, K16, 4.0, 1.0, tol=1e-7, max_iter=3000)
    assert b.L == pytest.approx(a.L / 2.0, rel=1e-4)
    assert b.K_norm == pytest.approx(a.K_norm, rel=1e-4)
    with pytest.raises(ValueError):
        rates.estimate_constants(fam, K16, 0.0, 1.0)
