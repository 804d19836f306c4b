"""Per-level CUDA-event times of the three step phases (adjoint / forward+SAGA /
image) of config D, for locating per-level overheads.

    python tools/phase_times.py [--config D] [--reps 20] [--world W --rank p]

With --world W the shard plan of rank p runs alone on this GPU (no collective).
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import _lib, ctmodel, mrsketch, solvers  # noqa: E402
from paper_2412_10249_b200 import dist as dist_mod  # noqa: E402
from paper_2412_10249_b200.synth import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="D")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--world", type=int, default=1, help="time rank --rank's shard of a world this size")
ap.add_argument("--rank", type=int, default=0)
args = ap.parse_args()
cfg = CONFIGS[args.config]
r = cfg.levels
geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
b = torch.randn(geom.m, device="cuda").double().cpu().numpy()
fam = mrsketch.make_family(r, cfg.side, [1.0 / r] * r, mode="coarse")
b = dist_mod.local_rows(geom, b, args.rank, args.world)
prob = dist_mod.make_sharded_problem(geom, b, fam, cfg.mu_g, rank=args.rank, world=args.world)
eng = prob.engine
st = solvers.init_state(prob, seed=1)
prm = solvers._params(1e-6, cfg.mu_g, cfg.mu_g)
L = _lib.lib()
h, s = eng.plan.handle, eng.plan.stream
cst = st.c_state(eng.b)
stream = torch.cuda.current_stream()


def timed(fn):
    for _ in range(3):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.reps)]
    for q in range(args.reps):
        ev[2 * q].record(stream)
        fn()
        ev[2 * q + 1].record(stream)
    torch.cuda.synchronize()
    return 1e3 * float(np.median([ev[2 * q].elapsed_time(ev[2 * q + 1]) for q in range(args.reps)]))


for lv in range(r):
    f = eng.plan.factors[lv]
    ta = timed(lambda: _lib.check(L.imask_step_adjoint(h, ctypes.byref(cst), lv, s)))
    tf = timed(lambda: _lib.check(L.imask_step_forward(h, ctypes.byref(cst), lv, ctypes.byref(prm), s)))
    ti = timed(lambda: _lib.check(L.imask_step_image(h, ctypes.byref(cst), lv, ctypes.byref(prm), s)))
    tall = timed(lambda: _lib.check(L.imask_sketch_step(h, ctypes.byref(cst), lv, ctypes.byref(prm), s)))
    n = cfg.side // f
    u = torch.rand(n * n, device="cuda")
    sino = torch.empty(eng.m_loc, device="cuda")
    tp = timed(lambda: eng.plan.project(u, f, sino))
    tb = timed(lambda: eng.plan.backproject(st.y, f, u))
    print(f"f={f:3d} adjoint {ta:8.1f}us forward {tf:8.1f}us image {ti:7.1f}us  step {tall:8.1f}us"
          f"  | project {tp:8.1f}us backproject {tb:8.1f}us", flush=True)
