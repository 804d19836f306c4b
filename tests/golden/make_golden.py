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
