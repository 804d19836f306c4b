"""Adjoint parity vs the float64 oracle at every factor of a few geometries
(relative L2 and max-abs / max-ref), for A/B runs of the adjoint variants
(e.g. IMASK_KNOT_MIN_F=2 to route factors >= 2 through the knot kernel).

    python tools/adj_parity.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ct_oracle  # noqa: E402
from paper_2412_10249_b200 import ctmodel  # noqa: E402

for side, na, nd, factors in ((256, 360, 363, (1, 2, 4, 8, 16, 32)), (48, 30, 70, (2, 3, 4, 6, 8, 12)),
                              (40, 17, None, (5, 8, 10)), (64, 90, 60, (8, 16))):
    geom = ctmodel.Geometry(side, na, nd)
    rng = np.random.default_rng(side)
    for f in factors:
        orc = ct_oracle.ProjectorOracle(side, na, geom.n_detectors, f)
        op = ctmodel.coarse_projector(geom, f)
        for kind in ("normal", "positive"):
            y = rng.standard_normal(orc.range_dim) if kind == "normal" else rng.random(orc.range_dim)
            got = op.adjoint_apply(torch.from_numpy(y.astype(np.float32)).cuda()).double().cpu().numpy()
            ref = orc.adjoint_apply(y.astype(np.float32).astype(np.float64))
            rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            mx = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
            print(f"{side}^2/{na}/{geom.n_detectors} f={f:2d} {kind:8s} rel {rel:.2e} max {mx:.2e}", flush=True)
