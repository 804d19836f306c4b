"""Fused engine against the generic device path (the same update through the
package's LinOp / ProxFn callables, reference state layout) on geometries up to
config E's size, where the float64 oracle's CSR no longer fits: sketch_step,
sketch_seq_step and the sharded phases. One-off hardening check."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import ctmodel, mrsketch, proxlib, solvers  # noqa: E402


def rel(a, b):
    return float(torch.linalg.norm(a.double() - b.double()) / (torch.linalg.norm(b.double()) + 1e-300))


cases = [(64, 90, 91, 3, 24), (200, 128, 283, 4, 16), (512, 720, 725, 5, 16), (1024, 360, 1449, 6, 14),
         (2048, 256, 2897, 7, 10), (1536, 180, 2173, 6, 8), (96, 120, 137, 6, 16), (272, 100, 385, 5, 12)]
for side, na, nd, r, iters in cases:
    probs = [1.0 / r] * r
    geom = ctmodel.Geometry(side, na, nd)
    gen = torch.Generator(device="cuda").manual_seed(side)
    b = torch.rand(geom.m, device="cuda", generator=gen) * side
    fam = mrsketch.make_family(r, side, probs, mode="coarse")
    K = ctmodel.projector_op(geom)
    pr = solvers.make_problem(K, b, fam, proxlib.ridge_fn(1e-2), proxlib.quadratic_conjugate_fn(b),
                              coarse_projector=lambda f: ctmodel.coarse_projector(geom, f))
    out = {}
    for name in ("fused", "generic", "seq_fused", "seq_generic"):
        seq = name.startswith("seq")
        st = (solvers.init_state(pr, seed=4) if name.endswith("fused")
              else solvers.init_state(pr, seed=4, ops=pr.ops))
        for _ in range(iters):
            if seq:
                solvers.sketch_seq_step(st, pr, 1e-6, 1e-2, 0.7)
            else:
                solvers.sketch_step(st, pr, 1e-6, 1e-2)
        torch.cuda.synchronize()
        out[name] = (st.x.clone(), st.y.clone())
    ex, ey = rel(out["fused"][0], out["generic"][0]), rel(out["fused"][1], out["generic"][1])
    sx, sy = rel(out["seq_fused"][0], out["seq_generic"][0]), rel(out["seq_fused"][1], out["seq_generic"][1])
    flag = "" if max(ex, ey, sx, sy) <= 1e-5 else "  <-- FAIL"
    print(f"side {side:5d} angles {na:4d} det {nd:5d} r {r} ({iters} its): sketch x {ex:.2e} y {ey:.2e} | "
          f"seq x {sx:.2e} y {sy:.2e}{flag}", flush=True)
    del pr, out
    torch.cuda.empty_cache()
