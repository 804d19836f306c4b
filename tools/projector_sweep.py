"""Projectors against the float64 oracle on stress geometries: detector counts
from half the image side to three times it, 1-3 angles, tiny and non-square-ish
grids, random unsorted angle subsets (no mirror layout), quad subsets, every
factor the side allows. One-off hardening check."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ct_oracle  # noqa: E402
from paper_2412_10249_b200 import ctmodel  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-300))


worst = 0.0
n_cases = 0
rng = np.random.default_rng(0)
for side in (1, 2, 6, 16, 36, 64, 100, 128, 192, 320):
    for na in (1, 2, 3, 8, 12, 50, 90, 180):
        for nd in sorted({max(1, side // 2), side, int(np.ceil(side * 2 ** 0.5)), 2 * side + 1, 3 * side + 2}):
            if side * side * na * nd > 6e8:
                continue
            geom = ctmodel.Geometry(side, na, nd)
            subsets = [None]
            if na >= 8:
                k = int(rng.integers(2, na))
                subsets.append(list(rng.permutation(na)[:k]))
            if na % 4 == 0 and na >= 12:
                subsets.append(list(ctmodel.quad_subset(na, [1, na // 4 - 1])))
            for sub in subsets:
                plan = ctmodel.Plan(geom, angles=sub) if sub is not None else ctmodel.Plan(geom)
                rows = na if sub is None else len(sub)
                f = 1
                while side % f == 0 and f <= side:
                    n = side // f
                    u = rng.random(n * n)
                    y = rng.standard_normal(rows * nd)
                    orc = ct_oracle.ProjectorOracle(side, na, nd, f, sub)
                    got_f = plan.project(torch.from_numpy(u.astype(np.float32)).cuda(), f).double().cpu().numpy()
                    got_a = plan.backproject(torch.from_numpy(y.astype(np.float32)).cuda(), f).double().cpu().numpy()
                    ref_f, ref_a = orc.apply(u), orc.adjoint_apply(y)
                    ef = rel(got_f, ref_f) if np.linalg.norm(ref_f) > 0 else float(np.abs(got_f).max())
                    ea = rel(got_a, ref_a) if np.linalg.norm(ref_a) > 0 else float(np.abs(got_a).max())
                    n_cases += 1
                    worst = max(worst, ef, ea)
                    if max(ef, ea) > 1.5e-5:
                        print(f"{"FAIL" if max(ef, ea) > 1e-4 else "note"} side {side} angles {na} det {nd} f {f} subset "
                              f"{'all' if sub is None else len(sub)}: forward {ef:.2e} adjoint {ea:.2e}", flush=True)
                    f *= 2
                del plan
    print(f"side {side}: {n_cases} cases, worst {worst:.2e}", flush=True)
print("worst", worst, "cases", n_cases)
