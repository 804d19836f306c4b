"""Per-rank step time of the angle-sharded ImaSk step at world sizes 1/2/4/8,
measured on ONE GPU (config D): each rank's shard plan runs its single-GPU step
graph (forward chain on the side stream, adjoint, image update) without the
all-reduce, so the numbers bound the multi-GPU step from below (the collective
is excluded, not emulated). Prints per-level times and the compute-only strong
scaling efficiency T1 / (W * max_rank T_W) of the level-averaged step.

    python tools/shard_probe.py [--worlds 1,2,4,8] [--reps 30]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import ctmodel, mrsketch, solvers  # noqa: E402
from paper_2412_10249_b200 import dist as dist_mod  # noqa: E402
from paper_2412_10249_b200.synth import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--all-ranks", action="store_true")
args = ap.parse_args()
cfg = CONFIGS["D"]
r = cfg.levels
geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
fam = mrsketch.make_family(r, cfg.side, [1.0 / r] * r, mode="coarse")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
b_full = torch.randn(geom.m, device=dev)
prm = solvers._params(1e-6, cfg.mu_g, cfg.mu_g)

results = {}
for W in [int(w) for w in args.worlds.split(",")]:
    per_rank = []
    for rank in (range(W) if args.all_ranks else sorted({0, W - 1})):
        idx = torch.as_tensor(ctmodel.shard_angles(geom.n_angles, rank, W), device=dev)
        b_loc = b_full.reshape(geom.n_angles, geom.n_detectors)[idx].reshape(-1).contiguous()
        prob = dist_mod.make_sharded_problem(geom, b_loc, fam, cfg.mu_g, rank=rank, world=W)
        eng = prob.engine
        st = solvers.init_state(prob, seed=1)
        L = solvers._lib.lib()
        times = []
        for lv in range(r):
            g, _ = eng.graph(st, lv, prm)
            for _ in range(3):
                solvers._lib.check(L.imask_graph_launch(g, eng.plan.stream))
            torch.cuda.synchronize()
            stream = torch.cuda.current_stream()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.reps)]
            for q in range(args.reps):
                flush.fill_(float(q))
                torch.cuda.synchronize()
                ev[2 * q].record(stream)
                solvers._lib.check(L.imask_graph_launch(g, eng.plan.stream))
                ev[2 * q + 1].record(stream)
            torch.cuda.synchronize()
            times.append(float(np.median([ev[2 * q].elapsed_time(ev[2 * q + 1])
                                          for q in range(args.reps)])) * 1e3)
        per_rank.append((rank, len(idx), times))
        eng.release_graphs()
        del prob, eng, st
        torch.cuda.empty_cache()
    worst = np.max([t for _, _, t in per_rank], axis=0)
    results[W] = worst
    for rank, rows, t in per_rank:
        print(f"W={W} rank {rank} ({rows} rows): " +
              "  ".join(f"f{2 ** (r - 1 - lv)} {t[lv]:7.1f}" for lv in range(r)) +
              f"  mean {np.mean(t):7.1f} us", flush=True)
T1 = np.mean(results[min(results)])
for W, t in results.items():
    print(f"W={W}: level-mean step {np.mean(t):7.1f} us (max over ranks), "
          f"compute-only efficiency {T1 / (W * np.mean(t)):.3f}  per level: " +
          " ".join(f"{results[min(results)][lv] / (W * t[lv]):.2f}" for lv in range(r)), flush=True)
