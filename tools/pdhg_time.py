"""Time device PDHG iterations (imask_pdhg_step) on config D."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import ctmodel, mrsketch, proxlib, solvers  # noqa: E402
from paper_2412_10249_b200.synth import CONFIGS, ellipse_phantom  # noqa: E402

cfg = CONFIGS["D"]
geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
K = ctmodel.projector_op(geom)
x_true = torch.from_numpy(ellipse_phantom(cfg.side, 0).astype(np.float32).ravel()).cuda()
b = K.apply(x_true)
fam = mrsketch.make_family(cfg.levels, cfg.side, [1.0 / cfg.levels] * cfg.levels, mode="coarse")
prob = solvers.make_problem(K, b, fam, proxlib.ridge_fn(cfg.mu_g), proxlib.quadratic_conjugate_fn(b),
                            coarse_projector=lambda f: ctmodel.coarse_projector(geom, f))
it = solvers._Pdhg(prob, *solvers.pdhg_parameters(1500.0, cfg.mu_g)[:3])
for _ in range(5):
    it.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 200
e0.record()
for _ in range(n):
    it.step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"PDHG config D: {ms:.3f} ms/iteration, {1e3 / ms:.1f} iter/s; 5000 iterations: {5 * ms:.2f} s")
