import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2412_10249_b200 import ctmodel
from oracle import ct_oracle
for side, na, nd in ((64, 90, 91), (256, 360, 363)):
    geom = ctmodel.Geometry(side, na, nd)
    plan = ctmodel.get_plan(geom)
    for f in (1, 2, 4):
        x = np.random.default_rng(0).random((side // f) ** 2)
        try:
            s = plan.project(torch.from_numpy(x.astype(np.float32)).cuda(), f)
            torch.cuda.synchronize()
            ref = ct_oracle.ProjectorOracle(side, na, nd, f).apply(x)
            err = np.linalg.norm(s.double().cpu().numpy() - ref) / np.linalg.norm(ref)
            print(side, f, "ok rel", err, flush=True)
        except Exception as e:
            print(side, f, "FAIL", e, flush=True)
            raise SystemExit(1)
