"""Break down bench.py's e2e leg (config D) into its host-visible phases."""
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
b_host = torch.randn(geom.m).pin_memory()
xref_host = torch.from_numpy(x_true).pin_memory()
dev = torch.device("cuda", 0)


def phase(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    print(f"{name:32s} {1e3 * (time.perf_counter() - t0):9.2f} ms", flush=True)
    return out


for rep in range(2):
    print(f"-- rep {rep}")
    b_dev = phase("h2d", lambda: b_host.to(dev, non_blocking=True))
    xref = xref_host.to(dev)
    prob = phase("make_sharded_problem", lambda: dist_mod.make_sharded_problem(geom, b_dev, fam, cfg.mu_g))
    st = phase("init_state", lambda: solvers.init_state(prob, seed=1))
    prm = solvers._params(1e-6, cfg.mu_g, cfg.mu_g)
    phase("graph capture x6", lambda: [prob.engine.graph(st, lv, prm) for lv in range(r)])
    sched = solvers.draw_levels(1, 0, 100, prob.cum_probs)
    phase("100 steps (no record)", lambda: [solvers._device_step(prob.engine, st, int(i), prm) for i in sched])
    phase("100 metrics", lambda: [solvers._metrics(st.x, xref) for _ in range(100)])
    prob.engine.release_graphs()
    phase("run(100, record_every=1)", lambda: solvers.run(prob, "sketch", 1e-6, cfg.mu_g, 100,
                                                         record_every=1, seed=1, x_ref=xref))
