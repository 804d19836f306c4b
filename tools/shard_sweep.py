"""Every shard of shard_angles over many angle counts and world sizes: its rows
equal the whole plan's rows, the shards' backprojections sum to the whole one,
at a full and a coarse level (contiguous, quad and block-cyclic shards; odd
counts; more ranks than quads). One-off hardening check."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import ctmodel  # noqa: E402


def rel(a, b):
    return float(torch.linalg.norm(a.double() - b.double()) / (torch.linalg.norm(b.double()) + 1e-300))


worst = 0.0
for side, nd in ((64, 91), (160, 227), (256, 363)):
    for na in (7, 9, 16, 30, 45, 61, 64, 100, 128, 180, 256, 360, 500, 512, 720, 1024):
        geom = ctmodel.Geometry(side, na, nd)
        full = ctmodel.Plan(geom)
        gen = torch.Generator(device="cuda").manual_seed(na)
        y = torch.randn(na, nd, device="cuda", generator=gen)
        for f in (1, 4):
            u = torch.rand((side // f) ** 2, device="cuda", generator=gen)
            s_full = full.project(u, f).reshape(na, nd).clone()
            b_full = full.backproject(y.reshape(-1), f).clone()
            for world in (2, 3, 4, 5, 8):
                if world > na:
                    continue
                acc = torch.zeros_like(b_full)
                e_rows = 0.0
                rows = 0
                for rank in range(world):
                    idx = list(ctmodel.shard_angles(na, rank, world))
                    rows += len(idx)
                    if not idx:
                        continue
                    plan = ctmodel.Plan(geom, angles=idx)
                    t = torch.as_tensor(idx, device="cuda")
                    part = plan.project(u, f).reshape(len(idx), nd)
                    e_rows = max(e_rows, rel(part, s_full[t]))
                    acc += plan.backproject(y[t].reshape(-1).contiguous(), f)
                    del plan
                e_bp = rel(acc, b_full)
                worst = max(worst, e_rows, e_bp)
                if rows != na or e_rows > 1e-6 or e_bp > 2e-6:
                    print(f"FAIL side {side} angles {na} f {f} world {world}: rows {rows} "
                          f"forward {e_rows:.2e} adjoint-sum {e_bp:.2e}", flush=True)
        del full
    print(f"side {side}: done, worst so far {worst:.2e}", flush=True)
print("worst", worst)
