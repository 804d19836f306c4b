mkdir -p gpurun_out
python bench.py --gpus 1 --steps 20 --warmup 5 --no-microbench --no-cpu-baseline > gpurun_out/b20.log 2>&1
python - > gpurun_out/mkprob_profile.log 2>&1 <<'P'
import cProfile, pstats, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2412_10249_b200 import ctmodel, mrsketch, solvers
from paper_2412_10249_b200 import dist as dist_mod
from paper_2412_10249_b200.synth import CONFIGS
cfg = CONFIGS["D"]; r = cfg.levels
geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
fam = mrsketch.make_family(r, cfg.side, [1.0 / r] * r, mode="coarse")
b = torch.randn(geom.m, device="cuda")
for _ in range(3): dist_mod.make_sharded_problem(geom, b, fam, cfg.mu_g)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): dist_mod.make_sharded_problem(geom, b, fam, cfg.mu_g)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
P
