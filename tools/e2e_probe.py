"""Break down bench.py's e2e leg (config D): host wall time of solvers.run vs the
device span its metric rows record, with and without per-step rows."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import ctmodel, mrsketch, solvers  # noqa: E402
from paper_2412_10249_b200 import dist as dist_mod  # noqa: E402
from paper_2412_10249_b200.synth import CONFIGS, ellipse_phantom  # noqa: E402

cfg = CONFIGS["D"]
r = cfg.levels
geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
fam = mrsketch.make_family(r, cfg.side, [1.0 / r] * r, mode="coarse")
x_true = ellipse_phantom(cfg.side, 0).astype(np.float32).ravel()
dev = torch.device("cuda", 0)
b = torch.randn(geom.m, device=dev)
xref = torch.from_numpy(x_true).to(dev)
prob = dist_mod.make_sharded_problem(geom, b, fam, cfg.mu_g)
prm = solvers._params(1e-6, cfg.mu_g, cfg.mu_g)
prob.engine.capture_all(solvers.init_state(prob, seed=1), prm)
solvers.run(prob, "sketch", 1e-6, cfg.mu_g, 5, record_every=1, seed=1, x_ref=xref)
for rec_every in (1, 1, 200, 200):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = solvers.run(prob, "sketch", 1e-6, cfg.mu_g, 200, record_every=rec_every, seed=1, x_ref=xref)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    span = rep.rows[-1][5] - rep.rows[0][5]
    print(f"record_every={rec_every:3d}: wall {1e3 * wall:7.2f} ms  device span k=0..200 "
          f"{1e3 * span:7.2f} ms  first row at {1e3 * rep.rows[0][5]:6.2f} ms", flush=True)
# the same 200 steps through the step graphs alone
st = solvers.init_state(prob, seed=1)
sched = solvers.draw_levels(1, 0, 200, prob.cum_probs)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in sched:
        solvers._device_step(prob.engine, st, int(i), prm)
    torch.cuda.synchronize()
    print(f"200 bare graph steps: {1e3 * (time.perf_counter() - t0):7.2f} ms", flush=True)
# host cost of re-targeting the cached step graphs to a new state's buffers
st2 = solvers.init_state(prob, seed=2)
torch.cuda.synchronize()
t0 = time.perf_counter()
for lv in range(r):
    prob.engine.graph(st2, lv, prm)
t1 = time.perf_counter()
for lv in range(r):
    prob.engine.graph(st2, lv, prm)
t2 = time.perf_counter()
print(f"re-target {r} step graphs to a new state: {1e3 * (t1 - t0):.2f} ms; "
      f"cached lookups: {1e3 * (t2 - t1):.3f} ms", flush=True)
