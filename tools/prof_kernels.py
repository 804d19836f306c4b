"""Launch the projector kernels of config D at every level (for ncu captures).

    python tools/prof_kernels.py [--levels 1,2,...] [--reps N]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import ctmodel  # noqa: E402
from paper_2412_10249_b200.synth import CONFIGS, ellipse_phantom  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="D")
ap.add_argument("--factors", default="1,2,4,8,16,32")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--world", type=int, default=1, help="rank --rank's angle shard of this world size")
ap.add_argument("--rank", type=int, default=0)
args = ap.parse_args()
cfg = CONFIGS[args.config]
geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
angles = ctmodel.shard_angles(geom.n_angles, args.rank, args.world) if args.world > 1 else None
plan = ctmodel.get_plan(geom, angles=angles) if angles is not None else ctmodel.get_plan(geom)
x = torch.from_numpy(ellipse_phantom(cfg.side, 0).astype(np.float32).ravel()).cuda()
y = torch.randn(plan.m_loc, device="cuda")
from paper_2412_10249_b200 import mrsketch  # noqa: E402

for f in [int(v) for v in args.factors.split(",")]:
    u = mrsketch.decimate(x.reshape(cfg.side, cfg.side), f).reshape(-1) if f > 1 else x
    for _ in range(args.reps):
        s = plan.project(u, f)
        b = plan.backproject(y, f)
    torch.cuda.synchronize()
    print(f"f={f} ok {float(s.abs().sum()):.4g} {float(b.abs().sum()):.4g}")
