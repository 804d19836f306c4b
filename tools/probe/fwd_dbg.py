import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2412_10249_b200 import ctmodel
geom = ctmodel.Geometry(64, 90, 91)
plan = ctmodel.get_plan(geom)
x = torch.rand(64 * 64, device="cuda")
s = plan.project(x, 1)
torch.cuda.synchronize()
print(s[:48].cpu().numpy().reshape(-1, 8))
