"""Per level: the step's forward phase (staging + projection + sinogram SAGA into
y_next) from one random x; y_next of every level saved to $OUT (debug aid for
staging path switches). Args: side n_angles n_det r"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import _lib, ctmodel, mrsketch, solvers  # noqa: E402
from paper_2412_10249_b200 import dist as dist_mod  # noqa: E402

side, na, nd, r = (int(v) for v in sys.argv[1:5])
geom = ctmodel.Geometry(side, na, nd)
b = np.random.default_rng(3).standard_normal(geom.m)
fam = mrsketch.make_family(r, side, [1.0 / r] * r, mode="coarse")
prob = dist_mod.make_sharded_problem(geom, b, fam, 1e-2)
st = solvers.init_state(prob, seed=4)
torch.manual_seed(0)
st.x.copy_(torch.rand(side * side, device="cuda"))
prm = solvers._params(2e-4, 1e-2, 1e-2)
h, s = prob.engine.plan.handle, prob.engine.plan.stream
out = {}
for lv in list(range(r)) + list(range(r)):
    cst = ctypes.byref(st.c_state(prob.engine.b))
    _lib.check(_lib.lib().imask_step_forward(h, cst, lv, ctypes.byref(prm), s))
    torch.cuda.synchronize()
    out[f"y{lv}"] = st.y_alt.cpu().numpy().copy()
np.savez(os.environ.get("OUT", "/tmp/stage.npz"), **out)
print("ok")
