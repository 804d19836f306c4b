"""One eager sketch_step per level on an angle-subset problem (debugging aid:
run under compute-sanitizer). Args: side n_angles n_det r [bases...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_10249_b200 import ctmodel, mrsketch, proxlib, solvers  # noqa: E402

side, na, nd, r = (int(v) for v in sys.argv[1:5])
bases = [int(v) for v in sys.argv[5:]] or [1, 2, 5, 17]
rows = ctmodel.quad_subset(na, bases)
geom = ctmodel.Geometry(side, na, nd)
b = np.random.default_rng(0).standard_normal(len(rows) * nd)
K = ctmodel.projector_op(geom, angles=rows)
fam = mrsketch.make_family(r, side, [1.0 / r] * r, mode="coarse")
prob = solvers.make_problem(K, b, fam, proxlib.ridge_fn(1e-2), proxlib.quadratic_conjugate_fn(b),
                            coarse_projector=lambda f: ctmodel.coarse_projector(geom, f, angles=rows))
prob.engine.use_graphs = False
print("rows", len(rows), "sym", prob.engine.plan.symmetric, "quad", prob.engine.plan.quad_forward,
      flush=True)
x = torch.rand(side * side, device="cuda")
for f in prob.engine.plan.factors:
    u = mrsketch.decimate(x.reshape(side, side), f).reshape(-1)
    y = ctmodel.coarse_projector(geom, f, angles=rows).apply(u)
    torch.cuda.synchronize()
    print("project f", f, float(y.norm()), flush=True)
    bp = ctmodel.coarse_projector(geom, f, angles=rows).adjoint_apply(y)
    torch.cuda.synchronize()
    print("backproject f", f, float(bp.norm()), flush=True)
st = solvers.init_state(prob, seed=1)
prm = prob.engine.params(1e-5, 1e-2)
for lv in range(r):
    solvers._device_step(prob.engine, st, lv, prm)
    torch.cuda.synchronize()
    print("step level", lv, float(st.x.norm()), flush=True)
