"""Where the fixed cost of bench.py's e2e leg goes at K = 20 (the driver's run):
PCIe copies, problem set-up, run()'s own start-up and read-back, each timed
with a synchronize on both sides."""
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
dev = torch.device("cuda", 0)
x_true = ellipse_phantom(cfg.side, 0).astype(np.float32).ravel()
b_host = torch.randn(geom.m).pin_memory()
xref_host = torch.from_numpy(x_true).pin_memory()
x_out = torch.empty(cfg.d).pin_memory()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20


def T(fn, reps=5):
    ts = []
    out = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return np.median(ts), out


ms, b_dev = T(lambda: b_host.to(dev, non_blocking=True))
print(f"H2D b ({b_host.numel() * 4 / 1e6:.1f} MB): {ms:.3f} ms = {b_host.numel() * 4 / ms / 1e6:.1f} GB/s")
ms, xr = T(lambda: xref_host.to(dev, non_blocking=True))
print(f"H2D x_ref ({xref_host.numel() * 4 / 1e6:.1f} MB): {ms:.3f} ms")
ms, _ = T(lambda: x_out.copy_(xr))
print(f"D2H x ({x_out.numel() * 4 / 1e6:.1f} MB): {ms:.3f} ms = {x_out.numel() * 4 / ms / 1e6:.1f} GB/s")
ms, prob = T(lambda: dist_mod.make_sharded_problem(geom, b_dev, fam, cfg.mu_g))
print(f"make_sharded_problem: {ms:.3f} ms")
prm = solvers._params(1e-6, cfg.mu_g, cfg.mu_g)
prob.engine.capture_all(solvers.init_state(prob, seed=2024), prm)
solvers.run(prob, "sketch", 1e-6, cfg.mu_g, K, record_every=1, seed=2024, x_ref=xr)
ms, rep = T(lambda: solvers.run(prob, "sketch", 1e-6, cfg.mu_g, K, record_every=1, seed=2024, x_ref=xr))
span = rep.rows[-1][5] - rep.rows[0][5]
print(f"run({K} steps, rows every step): {ms:.3f} ms; device span row 0 .. row {K}: {1e3 * span:.3f} ms")
ms, rep = T(lambda: solvers.run(prob, "sketch", 1e-6, cfg.mu_g, K, record_every=K, seed=2024, x_ref=xr))
print(f"run({K} steps, 2 rows): {ms:.3f} ms")
ms, rep = T(lambda: solvers.run(prob, "sketch", 1e-6, cfg.mu_g, 0, record_every=1, seed=2024, x_ref=xr))
print(f"run(0 steps): {ms:.3f} ms")
# pieces of run()'s start-up
ms, st = T(lambda: solvers.init_state(prob, seed=2024))
print(f"init_state: {ms:.3f} ms")
ms, rec = T(lambda: solvers._Recorder(xr, dev, K + 2, time.perf_counter()))
print(f"_Recorder(): {ms:.3f} ms")
ms, _ = T(lambda: solvers.draw_levels(2024, 0, K, prob.cum_probs))
print(f"draw_levels: {ms:.3f} ms")
ms, _ = T(lambda: (rep.x.clone(), rep.y.clone()))
print(f"x.clone(), y.clone(): {ms:.3f} ms")
