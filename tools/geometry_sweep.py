"""Sweep of unusual geometries (image sides that are not multiples of 32, odd /
non-quad angle counts, even and odd detector counts, every level count the side
allows): projections at every level and 12 solver iterations against the
float64 oracle (memory sums re-formed every 5 iterations), and a repeated
solve bit for bit. One-off hardening check."""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import solver_oracle as so  # noqa: E402
from paper_2412_10249_b200 import ctmodel, mrsketch, proxlib, solvers  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-300))


cases = [(48, 60, 69, 2), (40, 45, 57, 3), (72, 61, 103, 4), (80, 90, 114, 5), (96, 120, 137, 6),
         (112, 64, 159, 5), (144, 100, 205, 5), (176, 92, 250, 5), (136, 37, 193, 4),
         (200, 128, 283, 4), (24, 30, 35, 4), (12, 9, 17, 3), (160, 90, 227, 6), (192, 180, 272, 7)]
worst = 0.0
for side, na, nd, r in cases:
    probs = list(np.random.default_rng(side).dirichlet(np.ones(r) * 4.0))
    probs = [float(p) for p in np.asarray(probs) / np.sum(probs)]
    geom = ctmodel.Geometry(side, na, nd)
    rng = np.random.default_rng(3)
    x0 = rng.random(side * side)
    ops = so.SketchedCT(side, na, nd, probs)
    fam = mrsketch.make_family(r, side, probs, mode="coarse")
    errs = []
    for lev in range(1, r + 1):
        f = 2 ** (r - lev)
        u = rng.random((side // f) ** 2)
        y = rng.standard_normal(geom.m)
        P = ctmodel.coarse_projector(geom, f)
        errs.append(rel(P.apply(torch.from_numpy(u.astype(np.float32)).cuda()).double().cpu().numpy(),
                        ops.proj[f].apply(u)))
        errs.append(rel(P.adjoint_apply(torch.from_numpy(y.astype(np.float32)).cuda()).double().cpu().numpy(),
                        ops.proj[f].adjoint_apply(y)))
    b = ops.proj[1].apply(x0) + 0.01 * rng.standard_normal(geom.m)
    K = ctmodel.projector_op(geom)
    pr = solvers.make_problem(K, b, fam, proxlib.ridge_fn(1e-2), proxlib.quadratic_conjugate_fn(b),
                              coarse_projector=lambda f: ctmodel.coarse_projector(geom, f))
    runs = []
    for _ in range(2):
        st = solvers.init_state(pr, seed=9, resum_every=5)
        for _ in range(12):
            solvers.sketch_step(st, pr, 1e-4, 1e-2)
        runs.append((st.x.clone(), st.y.clone()))
    same = torch.equal(runs[0][0], runs[1][0]) and torch.equal(runs[0][1], runs[1][1])
    ost = so.init_state(ops, seed=9, resum_every=5)
    for _ in range(12):
        so.sketch_step(ost, ops, b, 1e-4, 1e-2, 1e-2)
    ex = rel(runs[0][0].double().cpu().numpy(), ost.x)
    ey = rel(runs[0][1].double().cpu().numpy(), ost.y)
    worst = max(worst, max(errs), ex, ey)
    flag = "" if (max(errs) <= 1e-4 and ex <= 1e-3 and ey <= 1e-3 and same) else "  <-- FAIL"
    print(f"side {side:4d} angles {na:4d} det {nd:4d} r {r}: projections {max(errs):.2e}  x {ex:.2e}  y {ey:.2e}  "
          f"repeat {'ok' if same else 'DIFFERS'}{flag}", flush=True)
print("worst", worst)
