"""Sketch operators (restriction, prolongation, every S_i including the
compensation S_r) against the float64 oracle over image sides and level
counts off the BASELINE grid. One-off hardening check."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import sketch_oracle  # noqa: E402
from paper_2412_10249_b200 import mrsketch  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-300))


worst = 0.0
for side in (8, 12, 20, 24, 40, 48, 72, 80, 96, 112, 144, 176, 200, 224, 272, 320, 1000, 1056):
    for r in range(1, 8):
        if side % (2 ** (r - 1)):
            continue
        rng = np.random.default_rng(side * 10 + r)
        probs = rng.dirichlet(np.ones(r) * 3.0)
        probs = [float(p) for p in probs / probs.sum()]
        x = rng.standard_normal((side, side))
        fam = mrsketch.make_family(r, side, probs, mode="coarse")
        xd = torch.from_numpy(x.astype(np.float32)).cuda()
        errs = []
        for i in range(1, r + 1):
            got = fam.apply_sketch(xd.reshape(-1), i).double().cpu().numpy().reshape(side, side)
            errs.append(rel(got, sketch_oracle.apply_sketch(x, probs, i)))
            f = 2 ** (r - i)
            if f > 1:
                low = mrsketch.decimate(xd, f)
                errs.append(rel(low.double().cpu().numpy(), sketch_oracle.decimate(x, f)))
                up = mrsketch.upsample(low, f)
                errs.append(rel(up.double().cpu().numpy(), sketch_oracle.upsample(sketch_oracle.decimate(x, f), f)))
        w = max(errs)
        worst = max(worst, w)
        if w > 1e-5:
            print(f"FAIL side {side} r {r}: {w:.2e} {['%.1e' % e for e in errs]}", flush=True)
print("worst", worst)
