L=paper_2412_10249_b200/libimask_b200.so
cp $L /tmp/lib_default.so; cp tools/variants/lib_bounds_selftest.so $L
python - > gpurun_out/bounds_selftest.log 2>&1 <<'P'
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2412_10249_b200 import _lib, ctmodel
geom = ctmodel.Geometry(1024, 1440, 1449)
plan = ctmodel.get_plan(geom)
out = (ctypes.c_ulonglong * 4)()
plan.project(torch.rand(1024 * 1024, device="cuda"), 1)
rc = _lib.lib().imask_debug_bounds(out, 1)
print("forward with the window limit tightened to kFWc - 40:", rc, list(out))
plan.backproject(torch.randn(plan.m_loc, device="cuda"), 1)
rc = _lib.lib().imask_debug_bounds(out, 1)
print("adjoint with the window limit tightened to W - 45:", rc, list(out))
P
cp /tmp/lib_default.so $L
