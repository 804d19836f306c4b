"""Host-side logic of the B200 path that needs no device: geometry tables, angle
slabs, sketch-family validation, synthetic inputs."""

import math

import numpy as np
import pytest

from oracle import ct_oracle
from paper_2412_10249_b200 import mrsketch
from paper_2412_10249_b200.ctmodel import Geometry, shard_angles, slab_bounds
from paper_2412_10249_b200.synth import CONFIGS, ellipse_phantom


def test_geometry_matches_reference_convention():
    g = Geometry(side=128, n_angles=180, n_detectors=183)
    assert g.m == 180 * 183
    assert np.array_equal(g.angles, ct_oracle.angles(180))
    assert np.array_equal(g.offsets, ct_oracle.offsets(183))
    assert Geometry(side=16, n_angles=20).n_detectors == 23


def test_snapped_axis_angles_exact():
    for n in (180, 360, 720, 1440, 2048):
        c, s = Geometry(side=64, n_angles=n).cos_sin()
        assert c[n // 2] == 0.0 and s[0] == 0.0
        assert c[0] == 1.0 and s[n // 2] == 1.0
        nonzero = np.ones(n, bool)
        nonzero[[0, n // 2]] = False
        assert np.all(c[nonzero] != 0.0) and np.all(s[nonzero] != 0.0)
        for a in (1, n // 3, n - 1):
            assert (c[a], s[a]) == ct_oracle.snapped_cos_sin(a * (math.pi / n))


@pytest.mark.parametrize("n,world", [(180, 8), (1440, 8), (7, 3), (2048, 2), (5, 1)])
def test_slabs_partition_angles(n, world):
    bounds = [slab_bounds(n, r, world) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == n
    for (b0, e0), (b1, e1) in zip(bounds, bounds[1:]):
        assert e0 == b1
    sizes = [e - b for b, e in bounds]
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("n,world", [(180, 8), (1440, 8), (1440, 3), (90, 4), (7, 3), (9, 2),
                                     (2048, 2), (5, 1), (6, 4)])
def test_shards_partition_angles_mirror_closed(n, world):
    shards = [shard_angles(n, r, world) for r in range(world)]
    flat = [a for sh in shards for a in sh]
    assert sorted(flat) == list(range(n))  # a partition of all angles
    sizes = [len(sh) for sh in shards]
    # balanced to the shard unit: 2 rows (mirror pairs), 4 (quads when n % 4 == 0)
    assert max(sizes) - min(sizes) <= (10 if n % 4 == 0 else 3)
    for rank, sh in enumerate(shards):
        # the row layout imask_plan_create_list turns into mirror-symmetric kernels:
        # [0 on rank 0] + rows i <-> s + n_loc - 1 - i holding a and n - a
        s0 = 1 if rank == 0 else 0
        assert (0 in sh) == (rank == 0) and (rank != 0 or sh[0] == 0)
        rows = sh[s0:]
        for i, a in enumerate(rows):
            assert rows[len(rows) - 1 - i] == n - a
        if n % 4 == 0 and n >= 8:
            # closed under the transpose a -> n/2 - a too (quad-mode forward)
            low = {a % (n // 2) for a in sh}
            assert all((n // 2 - a) % (n // 2) in low for a in low)


def test_family_validation_messages():
    with pytest.raises(ValueError, match="divisible"):
        mrsketch.make_family(4, 4, [0.25] * 4)
    with pytest.raises(ValueError, match="sum"):
        mrsketch.make_family(2, 8, [0.5, 0.6])
    with pytest.raises(ValueError, match="positive"):
        mrsketch.make_family(2, 8, [1.2, -0.2])
    with pytest.raises(ValueError, match="mode"):
        mrsketch.make_family(2, 8, [0.5, 0.5], mode="fancy")
    fam = mrsketch.make_family(4, 64, [0.25] * 4)
    assert fam.decim_factors == (8, 4, 2, 1)
    assert fam.factor(4) == 1
    with pytest.raises(ValueError, match="level 5 out of range 1..4"):
        fam.factor(5)
    assert [mrsketch.cost_fraction(fam, i) for i in (1, 2, 3, 4)] == [0.125, 0.25, 0.5, 1.0]


def test_synthetic_phantom_deterministic_and_clipped():
    a = ellipse_phantom(64, 3)
    b = ellipse_phantom(64, 3)
    assert np.array_equal(a, b)
    assert a.min() >= 0.0 and a.max() <= 1.0 and a.max() > 0.0
    assert not np.array_equal(a, ellipse_phantom(64, 4))


def test_epoch_iteration_counts():
    # E[dcost/iter] = 2 sum_i p_i / f_i: A 1.1667, D 0.65625
    assert CONFIGS["A"].iters_for_epochs() == math.ceil(20 / (2 * (1 / 3) * (1 / 4 + 1 / 2 + 1)))
    assert CONFIGS["D"].iters_for_epochs() == math.ceil(50 / 0.65625)


def test_pdhg_parameter_formulas():
    """test_solvers.py:258-271: ||K||^2 = 3 mu rho^2 gives kappa 2, sigma 1,
    tau 1/mu, theta 1/3; a zero norm is rejected."""
    from paper_2412_10249_b200.solvers import pdhg_parameters

    mu, rho = 2.0, 0.99
    sigma, tau, theta, kappa = pdhg_parameters(np.sqrt(3.0 * mu * rho ** 2), mu, rho)
    assert kappa == pytest.approx(2.0, rel=1e-12)
    assert sigma == pytest.approx(1.0, rel=1e-12)
    assert tau == pytest.approx(1.0 / mu, rel=1e-12)
    assert theta == pytest.approx(1.0 / 3.0, rel=1e-12)
    with pytest.raises(ValueError):
        pdhg_parameters(0.0, 1.0)
