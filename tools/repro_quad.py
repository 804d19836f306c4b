"""Quad-mode TMA forward vs the pair-mode kernels on one geometry (debug aid)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import ctmodel  # noqa: E402

side, na, nd = (int(v) for v in sys.argv[1:4])
f = int(sys.argv[4]) if len(sys.argv) > 4 else 1
geom = ctmodel.Geometry(side, na, nd)
plan = ctmodel.Plan(geom)
n = side // f
torch.manual_seed(0)
u = torch.rand(n * n, device="cuda")
s = plan.project(u, f)
torch.cuda.synchronize()
np.save(os.environ.get("OUT", "/tmp/out.npy"), s.cpu().numpy())
print("ok", float(s.abs().sum()))
