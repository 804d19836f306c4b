"""The angle-sharded step with a real NCCL process group of one rank, on one GPU:
CUDA-graph replays (adjoint, all-reduce, forward chain, image update captured
together) against the eager sharded step and the single-GPU step.

    python tools/sharded_graph_check.py   (prints one JSON line; used by tests)
"""
import json
import os
import socket
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import ctmodel, mrsketch, solvers  # noqa: E402
from paper_2412_10249_b200 import dist as dist_mod  # noqa: E402


def free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{free_port()}", rank=0,
                            world_size=1, device_id=dev)
    side, na, nd, probs, mu_g = 128, 180, 183, [0.25] * 4, 1e-2
    geom = ctmodel.Geometry(side, na, nd)
    b = np.random.default_rng(3).standard_normal(geom.m)
    fam = mrsketch.make_family(4, side, probs, mode="coarse")
    prm = solvers._params(2e-4, 1e-2, mu_g)
    runs, wall = {}, {}
    for name in ("single", "eager", "graph"):
        grp = None if name == "single" else dist.group.WORLD
        pr = dist_mod.make_sharded_problem(geom, b, fam, mu_g, 0, 1, grp)
        eng = pr.engine
        eng.use_graphs = name != "eager"
        st = solvers.init_state(pr, seed=5)
        sched = solvers.draw_levels(5, 0, 40, pr.cum_probs)
        launches = 0
        for lv in sched:
            launches += solvers._device_step(eng, st, int(lv), prm)
        torch.cuda.synchronize()
        runs[name] = (st.x.double().cpu().numpy(), st.y.double().cpu().numpy(), launches,
                      len(eng._sharded))
        # host-side cost of a step (wall clock over 200 more steps, one sync)
        t0 = time.perf_counter()
        for lv in solvers.draw_levels(5, 40, 200, pr.cum_probs):
            solvers._device_step(eng, st, int(lv), prm)
        torch.cuda.synchronize()
        wall[name] = round(1e6 * (time.perf_counter() - t0) / 200, 1)
    xs, ys = runs["single"][0], runs["single"][1]
    out = {
        "graph_eq_eager": bool(np.array_equal(runs["graph"][0], runs["eager"][0])
                               and np.array_equal(runs["graph"][1], runs["eager"][1])),
        "rel_x_vs_single": float(np.linalg.norm(runs["graph"][0] - xs) / np.linalg.norm(xs)),
        "rel_y_vs_single": float(np.linalg.norm(runs["graph"][1] - ys) / np.linalg.norm(ys)),
        "graphs_captured": runs["graph"][3],
        "launches": {k: v[2] for k, v in runs.items()},
        "wall_us_per_step": wall,
    }
    print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
