"""The product's angle-sharded solver in W processes on one GPU (gloo
all-reduce of the CUDA partial backprojections; gloo collectives are not
graph-capturable, so the eager sharded step runs). Launch with

    python -m torch.distributed.run --nproc-per-node W --master-addr 127.0.0.1 \\
        --master-port P tools/multiproc_check.py [--n-angles 180] [--iters 40]

Rank 0 also solves the unsharded problem on the same GPU and prints one JSON
line: x bit-identical across ranks, x / y against the single-GPU run.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import ctmodel, mrsketch, solvers  # noqa: E402
from paper_2412_10249_b200 import dist as dist_mod  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=128)
    ap.add_argument("--n-angles", type=int, default=180)
    ap.add_argument("--levels", type=int, default=4)
    ap.add_argument("--iters", type=int, default=40)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    side, na, r = args.side, args.n_angles, args.levels
    geom = ctmodel.Geometry(side, na)
    b = np.random.default_rng(3).standard_normal(geom.m)
    x_true = np.random.default_rng(4).random(side * side)
    fam = mrsketch.make_family(r, side, [1.0 / r] * r, mode="coarse")
    sigma, mu, mu_g = 2e-4, 1e-2, 1e-2
    prob = dist_mod.make_sharded_problem(geom, dist_mod.local_rows(geom, b, rank, world), fam,
                                         mu_g, rank, world, dist.group.WORLD)
    prob.engine.use_graphs = False
    rep = solvers.run(prob, "sketch", sigma, mu, args.iters, record_every=10, seed=5,
                      x_ref=x_true)
    x = rep.x.double().cpu()
    y = rep.y.double().cpu()
    xs = [torch.zeros_like(x) for _ in range(world)]
    dist.all_gather(xs, x)
    ys = [None] * world
    dist.all_gather_object(ys, y.numpy())
    rows = [rw[:3] for rw in rep.rows]
    all_rows = [None] * world
    dist.all_gather_object(all_rows, rows)
    if rank == 0:
        single = dist_mod.make_sharded_problem(geom, b, fam, mu_g)
        rep1 = solvers.run(single, "sketch", sigma, mu, args.iters, record_every=10, seed=5,
                           x_ref=x_true)
        x1 = rep1.x.double().cpu().numpy()
        y1 = rep1.y.double().cpu().numpy().reshape(na, geom.n_detectors)
        y_err = 0.0
        for p in range(world):
            idx = list(ctmodel.shard_angles(na, p, world))
            ref = y1[idx].ravel()
            y_err = max(y_err, float(np.linalg.norm(ys[p] - ref) / np.linalg.norm(ref)))
        out = {
            "world": world,
            "n_angles": na,
            "quad_shards": bool(prob.engine.plan.quad_forward),
            "x_identical_across_ranks": all(torch.equal(xs[0], t) for t in xs[1:]),
            "rows_identical_across_ranks": all(rw == all_rows[0] for rw in all_rows),
            "rel_x_vs_single": float(np.linalg.norm(xs[0].numpy() - x1) / np.linalg.norm(x1)),
            "rel_y_vs_single": y_err,
            "levels_match_single": [rw[:3] for rw in rep1.rows] == all_rows[0],
        }
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
