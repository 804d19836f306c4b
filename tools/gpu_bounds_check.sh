# The GPU test suite on the index-checked build (tools/variants/lib_bounds.so,
# built here first with `make -C paper_2412_10249_b200/csrc bounds`: -DIMASK_BOUNDS_CHECK=1): compute-sanitizer is closed on the pool, so
# the kernels' own range checks on every window / pair-image read stand in for
# memcheck. The session ends with "[bounds check] violations N".
mkdir -p gpurun_out
compute-sanitizer --version > gpurun_out/sanitizer_closed.log 2>&1
L=paper_2412_10249_b200/libimask_b200.so
cp $L /tmp/lib_default.so
cp tools/variants/lib_bounds.so $L
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/pytest_bounds.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bounds.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_bounds.log 2>&1
python - >> gpurun_out/pytest_bounds.log 2>&1 <<'P'
# the bench process's own count is not visible here; run config D and E projections at every level in this process
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2412_10249_b200 import _lib, ctmodel
from paper_2412_10249_b200.synth import CONFIGS
for key in ("D", "E"):
    cfg = CONFIGS[key]
    geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    for world, rank in ((1, 0), (8, 0), (8, 5)):
        angles = ctmodel.shard_angles(geom.n_angles, rank, world) if world > 1 else None
        plan = ctmodel.Plan(geom, angles=angles) if angles is not None else ctmodel.get_plan(geom)
        y = torch.randn(plan.m_loc, device="cuda")
        f = 1
        while f <= 2 ** (cfg.levels - 1):
            u = torch.rand((cfg.side // f) ** 2, device="cuda")
            plan.project(u, f); plan.backproject(y, f)
            f *= 2
out = (ctypes.c_ulonglong * 4)()
rc = _lib.lib().imask_debug_bounds(out, 0)
print(f"[bounds check] configs D and E, every level, whole set and two 1/8 shards: compiled in {rc}, violations {out[0]} (site {out[1]}, index {ctypes.c_longlong(out[2]).value}, limit {out[3]})")
P
# the geometries off the BASELINE grid (any-size sketch / image-side kernels), in one process
python - >> gpurun_out/pytest_bounds.log 2>&1 <<'P'
import ctypes, os, runpy, sys
sys.path.insert(0, os.getcwd())
runpy.run_path("tools/geometry_sweep.py", run_name="__main__")
from paper_2412_10249_b200 import _lib
out = (ctypes.c_ulonglong * 4)()
rc = _lib.lib().imask_debug_bounds(out, 0)
print(f"[bounds check] tools/geometry_sweep.py: compiled in {rc}, violations {out[0]} (site {out[1]}, index {ctypes.c_longlong(out[2]).value}, limit {out[3]})")
P
cp /tmp/lib_default.so $L
