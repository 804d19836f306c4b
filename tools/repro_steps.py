"""K fused sketch steps (step graphs) on one geometry, x and y saved to $OUT
(used by test_gpu_solver.py to compare path switches bit for bit).
Args: side n_angles n_det r K [world rank]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import ctmodel, mrsketch, solvers  # noqa: E402
from paper_2412_10249_b200 import dist as dist_mod  # noqa: E402

side, na, nd, r, K = (int(v) for v in sys.argv[1:6])
world, rank = (int(v) for v in sys.argv[6:8]) if len(sys.argv) > 7 else (1, 0)
geom = ctmodel.Geometry(side, na, nd)
b = np.random.default_rng(3).standard_normal(geom.m)
fam = mrsketch.make_family(r, side, [1.0 / r] * r, mode="coarse")
prob = dist_mod.make_sharded_problem(geom, dist_mod.local_rows(geom, b, rank, world), fam, 1e-2,
                                     rank, world)
prob.engine.shard = solvers.Shard()  # the phases on one GPU, no collective
st = solvers.init_state(prob, seed=4)
torch.manual_seed(0)
st.x.copy_(torch.rand(side * side, device="cuda"))
prm = solvers._params(1e-6, 1e-2, 1e-2)
levels = list(range(r)) * 2 + [int(v) for v in solvers.draw_levels(4, 0, K, prob.cum_probs)]
for lv in levels:
    solvers._device_step(prob.engine, st, lv, prm)
torch.cuda.synchronize()
np.savez(os.environ.get("OUT", "/tmp/steps.npz"), x=st.x.cpu().numpy(), y=st.y.cpu().numpy())
print("ok", float(st.x.abs().sum()))
