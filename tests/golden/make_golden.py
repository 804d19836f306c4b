"""Generate the golden fixtures of tests/golden/ from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package `mrtomo` read-only from
/root/reference/pkg/src and records its outputs on seeded inputs. The GPU box
has no /root/reference: the committed .npz files are what the oracle and the
CUDA path are checked against there.

Fixtures:
  rng.npz      draw_level sequences / uniform_at values      (solvers.py:30-48)
  proj_small.npz ray_matrix CSR of small geometries incl. coarse pixel widths,
               odd and even detector counts                  (ctmodel.py:73-154)
  proj_A.npz   config A (128^2 / 180 / 183): coarse_projector(geom, f).apply /
               adjoint_apply at f = 1, 2, 4 on the seeded ellipse phantom and
               a seeded sinogram                              (ctmodel.py:194-204)
  proj_D_sampled.npz  config D (1024^2 / 1440 / 1449) on sampled angles
               {0, 1, 359, 360, 719, 720, 721, 1439} at f = 1 and 32 via
               ray_matrix (Kx rows, and K^T y at 4096 sampled pixels)
  sketch.npz   decimate / upsample / SketchFamily.apply_sketch (mrsketch.py)
  tv.npz       prox_tv_nonneg (proxlib.py:102-148) on seeded images: 50
               inner iterations (the default) and a 4x4 step image at 4000
  solver_A.npz sketch_step trajectory on config A (coarse mode, ridge
               mu_g = 1e-2, sigma = 3e-5, mu = mu_g): x, y, sums after
               18 iterations (= 20 epochs) and after 200 iterations
  solver_A_long.npz  config A, 1100 iterations at sigma = 1e-5 (stable; a
               1e-7 perturbation of b grows to ~3e-7 by k = 1100): x, y,
               sums at k = 999, 1000 (after the resum of solvers.py:219-220)
               and 1100
  solver_C.npz sketch_step on config C (512^2 / 720 / 725, r = 5, uniform
               probs, sigma = 2.5e-6): x, y after 26 and 52 iterations
               (52 = 40 epochs); b is rounded to float32 before the run, so
               both sides see identical data
  solver_D_subset.npz  sketch_step at the D grid (1024^2, 6 levels, 1449
               bins) on a quad-closed subset of 64 of the 1440 angles (rows
               in the layout ctmodel.quad_subset returns): the reference
               solver on LinOps built from ray_matrix on those rows, 77
               iterations (= 50 epochs), sigma = 5e-6
  proj_C_sampled.npz / proj_E_sampled.npz  configs C and E on sampled
               angles (incl. theta = 0, pi/4, pi/2 and their neighbours) at
               every level factor: forward rows of the decimated phantom and
               the adjoint of a seeded sinogram on those rows (at 4096 sampled
               pixels on fine grids, whole images on coarse ones)
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from mrtomo import ctmodel, mrsketch, proxlib, solvers  # noqa: E402

from paper_2412_10249_b200.synth import CONFIGS, add_gaussian_noise, ellipse_phantom  # noqa: E402

SIGMA_A = 3e-5
ITERS_A = (18, 200)
D_ANGLES = np.array([0, 1, 359, 360, 719, 720, 721, 1439])


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def gen_rng():
    out = {}
    prob_sets = {
        "u3": [1 / 3] * 3,
        "u6": [1 / 6] * 6,
        "p4": [0.3, 0.3, 0.2, 0.2],
        "u7": [1 / 7] * 7,
    }
    seeds = [0, 7, 12345, 2**63 + 5, 2**64 - 1]
    for pname, p in prob_sets.items():
        cum = np.cumsum(p)
        for si, seed in enumerate(seeds):
            out[f"levels_{pname}_s{si}"] = np.array(
                [solvers.draw_level(seed, k, cum) for k in range(5000)], dtype=np.int8
            )
    out["seeds"] = np.array([str(s) for s in seeds])
    out["uniform_s12345"] = np.array([solvers.uniform_at(12345, k) for k in range(256)])
    save("rng.npz", **out)


def gen_proj_small():
    out = {}
    cases = [(16, 20, 23, 1), (16, 20, 23, 2), (32, 36, 47, 1), (32, 36, 47, 4),
             (32, 36, 46, 2), (8, 15, None, 1), (64, 90, 91, 8), (16, 7, 23, 1)]
    for idx, (side, na, nd, f) in enumerate(cases):
        g = ctmodel.Geometry(side, na, nd)
        mat = ctmodel.ray_matrix(side // f, float(f), g.angles, g.offsets)
        out[f"c{idx}_meta"] = np.array([side, na, g.n_detectors, f])
        out[f"c{idx}_data"] = mat.data
        out[f"c{idx}_indices"] = mat.indices
        out[f"c{idx}_indptr"] = mat.indptr
    save("proj_small.npz", **out)


def gen_proj_A():
    cfg = CONFIGS["A"]
    g = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    x = ellipse_phantom(cfg.side, 0)
    rng = np.random.default_rng(20240817)
    y = rng.standard_normal(g.m)
    out = {"x": x}
    out["y"] = y
    for f in (1, 2, 4):
        op = ctmodel.coarse_projector(g, f)
        xl = mrsketch.decimate(x, f).ravel()
        out[f"fwd_f{f}"] = op.apply(xl)
        out[f"adj_f{f}"] = op.adjoint_apply(y)
    save("proj_A.npz", **out)


def gen_proj_D_sampled():
    cfg = CONFIGS["D"]
    g = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    x = ellipse_phantom(cfg.side, 0)
    rng = np.random.default_rng(7)
    ys = rng.standard_normal(len(D_ANGLES) * g.n_detectors)
    pix = np.sort(rng.choice(cfg.side * cfg.side, size=4096, replace=False))
    out = {"angles": D_ANGLES, "y": ys, "pix": pix}
    for f in (1, 32):
        mat = ctmodel.ray_matrix(cfg.side // f, float(f), g.angles[D_ANGLES], g.offsets)
        xl = mrsketch.decimate(x, f).ravel()
        out[f"fwd_f{f}"] = mat @ xl
        bp = mat.T @ ys
        if f == 1:
            out[f"adj_f{f}_at_pix"] = bp[pix]
        else:
            out[f"adj_f{f}"] = bp
    for f in (2, 4, 8, 16):  # the intermediate levels (sampled pixels on the fine grids)
        low = cfg.side // f
        mat = ctmodel.ray_matrix(low, float(f), g.angles[D_ANGLES], g.offsets)
        out[f"fwd_f{f}"] = mat @ mrsketch.decimate(x, f).ravel()
        bp = mat.T @ ys
        if low * low > 65536:
            pf = np.sort(rng.choice(low * low, size=4096, replace=False))
            out[f"pix_f{f}"] = pf
            out[f"adj_f{f}"] = bp[pf]
        else:
            out[f"adj_f{f}"] = bp
    save("proj_D_sampled.npz", **out)


def gen_sketch():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((64, 64))
    out = {"x": x}
    for f in (2, 4, 8):
        out[f"dec_f{f}"] = mrsketch.decimate(x, f)
        out[f"up_f{f}"] = mrsketch.upsample(mrsketch.decimate(x, f), f)
    for name, probs in (("u3", [1 / 3] * 3), ("p4", [0.3, 0.3, 0.2, 0.2]), ("u6", [1 / 6] * 6)):
        fam = mrsketch.make_family(len(probs), 64, probs)
        for i in range(1, fam.r + 1):
            out[f"S_{name}_{i}"] = fam.apply_sketch(x.ravel(), i)
    save("sketch.npz", **out)


def gen_solver_A():
    cfg = CONFIGS["A"]
    g = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    K = ctmodel.projector_op(g)
    x_true = ellipse_phantom(cfg.side, 0)
    sino = K.apply(x_true.ravel())
    b = add_gaussian_noise(sino, cfg.kappa, 1)
    r = cfg.levels
    fam = mrsketch.make_family(r, cfg.side, [1.0 / r] * r, mode="coarse")
    prob = solvers.make_problem(
        K, b, fam, proxlib.ridge_fn(cfg.mu_g), proxlib.quadratic_conjugate_fn(b),
        coarse_projector=lambda f: ctmodel.coarse_projector(g, f),
    )
    st = solvers.init_state(prob, seed=11)
    out = {"b": b, "x_true": x_true.ravel(), "sigma": SIGMA_A, "mu": cfg.mu_g, "seed": 11}
    levels = []
    for k in range(1, max(ITERS_A) + 1):
        solvers.sketch_step(st, prob, SIGMA_A, cfg.mu_g)
        levels.append(st.last_level)
        if k in ITERS_A:
            out[f"x_{k}"] = st.x.copy()
            out[f"y_{k}"] = st.y.copy()
            out[f"phi_sum_{k}"] = st.phi_sum.copy()
            out[f"psi_sum_{k}"] = st.psi_sum.copy()
            out[f"cost_{k}"] = st.cost
    out["levels"] = np.array(levels, dtype=np.int8)
    save("solver_A.npz", **out)


def _ref_problem(side, n_det, angles_rows, n_angles, b, r, mu_g):
    """Reference coarse-mode ridge problem whose operators are ray_matrix on the
    given angle rows (the reference's own Siddon matrices and solver)."""
    from mrtomo import linops

    g = ctmodel.Geometry(side, n_angles, n_det)
    th = g.angles[np.asarray(angles_rows)]

    def op(f):
        mat = ctmodel.ray_matrix(side // f, float(f), th, g.offsets)
        mt = mat.T.tocsr()
        return linops.LinOp(mat.shape[1], mat.shape[0], lambda x, m=mat: m @ x,
                            lambda y, m=mt: m @ y)

    K = op(1)
    fam = mrsketch.make_family(r, side, [1.0 / r] * r, mode="coarse")
    prob = solvers.make_problem(K, b, fam, proxlib.ridge_fn(mu_g), proxlib.quadratic_conjugate_fn(b),
                                coarse_projector=op)
    return K, prob


def _trajectory(prob, sigma, mu, seed, stops, extra=()):
    st = solvers.init_state(prob, seed=seed)
    out, levels = {}, []
    for k in range(1, max(stops) + 1):
        solvers.sketch_step(st, prob, sigma, mu)
        levels.append(st.last_level)
        if k in stops:
            out[f"x_{k}"] = st.x.astype(np.float32)
            out[f"y_{k}"] = st.y.astype(np.float32)
            out[f"cost_{k}"] = st.cost
            for name in extra:
                out[f"{name}_{k}"] = getattr(st, name).astype(np.float32)
    out["levels"] = np.array(levels, dtype=np.int8)
    return out


def gen_solver_A_long():
    cfg = CONFIGS["A"]
    g = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    K = ctmodel.projector_op(g)
    b = add_gaussian_noise(K.apply(ellipse_phantom(cfg.side, 0).ravel()), cfg.kappa, 1)
    b = b.astype(np.float32).astype(float)
    fam = mrsketch.make_family(3, cfg.side, [1.0 / 3] * 3, mode="coarse")
    prob = solvers.make_problem(K, b, fam, proxlib.ridge_fn(cfg.mu_g),
                                proxlib.quadratic_conjugate_fn(b),
                                coarse_projector=lambda f: ctmodel.coarse_projector(g, f))
    out = _trajectory(prob, 1e-5, cfg.mu_g, 5, (999, 1000, 1100), ("phi_sum", "psi_sum"))
    save("solver_A_long.npz", b=b.astype(np.float32), sigma=1e-5, mu=cfg.mu_g, seed=5, **out)


def gen_solver_C():
    cfg = CONFIGS["C"]
    g = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    K = ctmodel.projector_op(g)
    b = add_gaussian_noise(K.apply(ellipse_phantom(cfg.side, 0).ravel()), cfg.kappa, 1)
    b = b.astype(np.float32).astype(float)
    fam = mrsketch.make_family(cfg.levels, cfg.side, [1.0 / cfg.levels] * cfg.levels,
                               mode="coarse")
    prob = solvers.make_problem(K, b, fam, proxlib.ridge_fn(cfg.mu_g),
                                proxlib.quadratic_conjugate_fn(b),
                                coarse_projector=lambda f: ctmodel.coarse_projector(g, f))
    out = _trajectory(prob, 2.5e-6, cfg.mu_g, 17, (26, cfg.iters_for_epochs()))
    save("solver_C.npz", b=b.astype(np.float32), sigma=2.5e-6, mu=cfg.mu_g, seed=17, **out)


D_SUBSET_BASES = (1, 2, 5, 17, 44, 89, 120, 150, 179, 211, 250, 301, 333, 358, 359)


def gen_solver_D_subset():
    from paper_2412_10249_b200.ctmodel import quad_subset

    cfg = CONFIGS["D"]
    rows = quad_subset(cfg.n_angles, D_SUBSET_BASES)
    assert len(rows) == 64
    x_true = ellipse_phantom(cfg.side, 0).ravel()
    g = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    mat = ctmodel.ray_matrix(cfg.side, 1.0, g.angles[np.asarray(rows)], g.offsets)
    b = add_gaussian_noise(mat @ x_true, cfg.kappa, 1).astype(np.float32).astype(float)
    del mat
    _, prob = _ref_problem(cfg.side, cfg.n_det, rows, cfg.n_angles, b, cfg.levels, cfg.mu_g)
    out = _trajectory(prob, 5e-6, cfg.mu_g, 23, (cfg.iters_for_epochs(),))
    save("solver_D_subset.npz", rows=np.asarray(rows), bases=np.asarray(D_SUBSET_BASES),
         b=b.astype(np.float32), sigma=5e-6, mu=cfg.mu_g, seed=23, **out)


def _proj_sampled(cfg, sel, name):
    g = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    x = ellipse_phantom(cfg.side, 0)
    rng = np.random.default_rng(11)
    ys = rng.standard_normal(len(sel) * g.n_detectors)
    out = {"angles": np.asarray(sel), "y": ys.astype(np.float32)}
    ysf = ys.astype(np.float32).astype(float)
    for lv in range(cfg.levels):
        f = 2 ** lv
        low = cfg.side // f
        mat = ctmodel.ray_matrix(low, float(f), g.angles[np.asarray(sel)], g.offsets)
        xl = mrsketch.decimate(x, f).ravel() if f > 1 else x.ravel()
        out[f"fwd_f{f}"] = mat @ xl
        bp = mat.T @ ysf
        if low * low > 65536:
            pix = np.sort(rng.choice(low * low, size=4096, replace=False))
            out[f"pix_f{f}"] = pix
            out[f"adj_f{f}"] = bp[pix]
        else:
            out[f"adj_f{f}"] = bp
        del mat
    save(name, **out)


def gen_proj_C_sampled():
    _proj_sampled(CONFIGS["C"], [0, 1, 179, 180, 181, 359, 360, 361, 540, 719], "proj_C_sampled.npz")


def gen_proj_E_sampled():
    _proj_sampled(CONFIGS["E"], [0, 1, 511, 512, 1023, 1024, 1025, 1536, 2047],
                  "proj_E_sampled.npz")


def gen_proj_width():
    """project / backproject with pixel_width != 1 (ctmodel.py:170-191)."""
    out = {}
    rng = np.random.default_rng(5)
    cases = [(16, 20, 23, 0.5), (16, 20, 23, 1.5), (32, 36, 47, 2.0), (16, 24, 23, 0.25),
             (24, 28, 35, 3.0), (16, 20, 22, 0.75)]
    for idx, (side, na, nd, h) in enumerate(cases):
        g = ctmodel.Geometry(side, na, nd)
        x = rng.standard_normal(side * side)
        y = rng.standard_normal(g.m)
        out[f"c{idx}_meta"] = np.array([side, na, nd, h])
        out[f"c{idx}_x"] = x
        out[f"c{idx}_y"] = y
        out[f"c{idx}_fwd"] = ctmodel.project(g, x.reshape(side, side), pixel_width=h).ravel()
        out[f"c{idx}_adj"] = ctmodel.backproject(g, y.reshape(na, nd), pixel_width=h).ravel()
    save("proj_width.npz", **out)


RATE_CASES = ((1492.0, 861.3, 1492.0, 1 / 3), (2.0, 1.5, 3.0, 0.25), (5.0, 3.0, 6.0, 0.1),
              (1.0, 1.0, 1.0, 1.0), (40.0, 10.0, 35.0, 0.2))


def gen_rates():
    """Step-size theory of rates.py:122-301 on fixed constants (scalar host math)."""
    from mrtomo import rates

    out = {"cases": np.array(RATE_CASES)}
    for idx, (L, Lb, Lbp, mp) in enumerate(RATE_CASES):
        rc = rates.RateConstants(L=L, Lbar=Lb, Lbar_p=Lbp, min_p=mp, mu_g=1.0, mu_fstar=1.0)
        rows = []
        c_bar = 1.0 / (1.0 + (L * 1.01) ** 2 + (Lbp * 1.01) ** 2)
        for cf in (1e-3, 0.1, 0.5, 0.9):
            for rho in (0.05, 0.5, 0.95):
                pl = rates.plan_for(rc, cf * c_bar, rho)
                lo, hi = rates.admissible_interval(pl)
                rows.append([pl.a, pl.b, pl.c, pl.c_bar, pl.rho, pl.alpha, pl.eta_star,
                             pl.sigma_star, pl.theta_star, lo, hi,
                             float(pl.theta_of(0.5 * pl.eta_star))])
        out[f"plans_{idx}"] = np.array(rows)
        best = rates.optimal_step(rc)
        free = rates.optimal_step(rc, rho=None, num_c=25, num_rho=20)
        out[f"opt_{idx}"] = np.array([[p.c, p.rho, p.eta_star, p.sigma_star, p.theta_star]
                                      for p in (best, free)])
        grid = rates.step_plan_grid(rc, num_c=7, num_rho=5)
        out[f"grid_{idx}"] = np.array([[p.c, p.rho, p.theta_star] for p in grid])
        out[f"base_{idx}"] = np.array([rates.sigma_baseline(L, Lb)])
        out[f"unnorm_{idx}"] = np.array([rates.theta_unnormalized(s, mu, L, Lbp, Lb, mp, a, b)
                                         for s, mu, a, b in ((1e-3, 1.0, 2.0, 0.5),
                                                             (0.2, 0.1, 0.7, 3.0))])
    save("rates.npz", **out)


def gen_tv():
    out = {}
    rng = np.random.default_rng(21)
    for side, sigma, mu_g in ((16, 0.8, 0.5), (40, 0.3, 1.0), (64, 1.0, 0.25)):
        xp = rng.standard_normal(side * side) * 0.5 + 0.3
        out[f"xp_{side}"] = xp
        out[f"out_{side}"] = proxlib.prox_tv_nonneg(xp, sigma, mu_g)
        out[f"par_{side}"] = np.array([sigma, mu_g])
    img = np.zeros((4, 4))
    img[:, 2:] = 1.0
    img[1, 1] = -0.3
    out["xp_step"] = img.ravel()
    out["out_step"] = proxlib.prox_tv_nonneg(img.ravel(), 0.8, 0.5, inner_iters=4000,
                                             inner_tol=1e-13)
    save("tv.npz", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # e.g. `make_golden.py tv`: one fixture
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        sys.exit(0)
    gen_tv()
    gen_rng()
    gen_proj_small()
    gen_sketch()
    gen_proj_A()
    gen_solver_A()
    gen_proj_D_sampled()
