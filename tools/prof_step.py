"""One eager sketch_step per listed level of config D (for ncu captures of the
kernels of a step: forward chain, adjoint, image update).

    python tools/prof_step.py [--levels 5,4,0]   (0-based level index; 5 = f=1 for r=6)
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import ctmodel, mrsketch, solvers  # noqa: E402
from paper_2412_10249_b200 import dist as dist_mod  # noqa: E402
from paper_2412_10249_b200.synth import CONFIGS, ellipse_phantom  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="D")
ap.add_argument("--levels", default="5,4,0")
args = ap.parse_args()
cfg = CONFIGS[args.config]
r = cfg.levels
geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
plan = ctmodel.get_plan(geom)
x_true = torch.from_numpy(ellipse_phantom(cfg.side, 0).astype(np.float32).ravel()).cuda()
b = plan.project(x_true, 1)
fam = mrsketch.make_family(r, cfg.side, [1.0 / r] * r, mode="coarse")
prob = dist_mod.make_sharded_problem(geom, b, fam, cfg.mu_g)
eng = prob.engine
eng.use_graphs = False
st = solvers.init_state(prob, seed=1, x0=x_true)
prm = solvers._params(1e-6, cfg.mu_g, cfg.mu_g)
for lv in [int(v) for v in args.levels.split(",")]:
    solvers._device_step(eng, st, lv, prm)
torch.cuda.synchronize()
print("ok", float(st.x.abs().sum()))
