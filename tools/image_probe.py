"""Image-side SAGA kernels (imask_step_image) on config D, timed alone: one cold
launch between CUDA events (bench.py's hbm_kernels figure) and back to back
over rotating buffer sets larger than L2 (events around the batch).

    python tools/image_probe.py [--levels 5,0] [--sets 12]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10249_b200 import _lib, ctmodel, mrsketch, solvers  # noqa: E402
from paper_2412_10249_b200 import dist as dist_mod  # noqa: E402
from paper_2412_10249_b200.synth import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--levels", default="5,4,0")
ap.add_argument("--sets", type=int, default=12)
args = ap.parse_args()
cfg = CONFIGS["D"]
r = cfg.levels
geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
fam = mrsketch.make_family(r, cfg.side, [1.0 / r] * r, mode="coarse")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
sink = torch.empty((), device=dev)
b = torch.randn(geom.m, device=dev)
prob = dist_mod.make_sharded_problem(geom, b, fam, cfg.mu_g, rank=0, world=1)
eng = prob.engine
st = solvers.init_state(prob, seed=1)
prm = solvers._params(1e-6, cfg.mu_g, cfg.mu_g)
L = _lib.lib()
plan = eng.plan
stream = torch.cuda.current_stream()
sets = []
for _ in range(args.sets):
    bufs = [torch.zeros(cfg.d, device=dev) for _ in range(3)] + [torch.zeros(st.phi_tab.numel(), device=dev)]
    cs = _lib.ImaskState(bufs[0].data_ptr(), st.y.data_ptr(), eng.b.data_ptr(), bufs[1].data_ptr(),
                         st.psi_sum.data_ptr(), bufs[3].data_ptr(), st.psi_tab.data_ptr(),
                         bufs[2].data_ptr(), None, None)
    sets.append((bufs, cs))
peak = 6546.9
for lv in [int(v) for v in args.levels.split(",")]:
    f = 2 ** (r - 1 - lv)
    nbytes = 4.0 * 7 * cfg.d if f == 1 else 4.0 * (4 * cfg.d + 3 * cfg.d // (f * f))
    cold = []
    for q in range(25):
        sink.copy_(flush.sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.check(L.imask_step_image(plan.handle, ctypes.byref(sets[q % len(sets)][1]), lv,
                                      ctypes.byref(prm), plan.stream))
        e1.record(stream)
        torch.cuda.synchronize()
        if q >= 5:
            cold.append(e0.elapsed_time(e1))
    b2b = []
    for q in range(8):
        sink.copy_(flush.sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _, cs in sets:
            _lib.check(L.imask_step_image(plan.handle, ctypes.byref(cs), lv, ctypes.byref(prm),
                                          plan.stream))
        e1.record(stream)
        torch.cuda.synchronize()
        if q >= 2:
            b2b.append(e0.elapsed_time(e1) / len(sets))
    c, bb = float(np.mean(cold)) * 1e3, float(np.median(b2b)) * 1e3
    print(f"f={f:2d}  cold {c:6.2f} us {nbytes / c / 1e3:6.0f} GB/s ({nbytes / c / 1e3 / peak:.3f})"
          f"  back-to-back {bb:6.2f} us {nbytes / bb / 1e3:6.0f} GB/s ({nbytes / bb / 1e3 / peak:.3f})",
          flush=True)
