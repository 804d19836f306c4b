"""ImaSk hot-path benchmark on B200 (config D: 1024^2, 1440 angles, 1449 bins, r = 6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

A step is one parallel ImaSk iteration (sketch_step, solvers.py:194-221) at the
level drawn by the reference's counter-based RNG for that iteration: the
adjoint of level i on y^k, the forward of level i on x^k fused with the
sinogram-side SAGA update, and the image-side update. With N > 1 (torchrun)
angles are sharded and the partial backprojection is all-reduced over NCCL.

value   = iterations/s of the whole job (device time, CUDA events per step on
          the launching stream, L2 flushed between steps, max over ranks).
e2e     = iterations/s through the public API solvers.run(..., record_every=1,
          x_ref=...) from host data: b copied from pinned host memory inside the
          timed region, per-iteration metric read-back (the reference run()'s
          rel_dist / psnr row), final x copied back.
roofline = the dominant kernel (the slower level-1 projector) against measured
          HBM bandwidth on its algorithmic bytes, plus an FP32-issue view (footprint
          evaluations/s against a live FFMA-chain peak) and the HBM-bound
          image-side SAGA kernels against HBM bandwidth (hbm_kernels).
cpu_baseline / --impl reference = the reference algorithm (scipy CSR float64,
          oracle/ restatement) on a sampled-angle slice of config D, scaled to
          the full angle count (the full CSR needs ~130 GB), its CSR
          matvecs split over every host core the process may use.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIG_KEY = "D"
SEED = 2024
SIGMA = 1e-6  # explicit step (theory sigma* ~ 1e-7 at raw ||K||; any positive value times the same)
CPU_SAMPLE_ANGLES = 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--config", default=CONFIG_KEY)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-microbench", action="store_true",
                    help="skip the projector microbenchmark (config E)")
    ap.add_argument("--collective", action="store_true",
                    help="run the angle-sharded (NCCL) step path even at one rank (path check)")
    ap.add_argument("--no-full-reference", action="store_true",
                    help="--impl reference: skip the fully timed config-C reference solve")
    ap.add_argument("--steps-only", action="store_true",
                    help="skip the post-run kernel measurements (launch-list profiling runs)")
    return ap.parse_args()


# ---------------------------------------------------------------- reference arm

def ray_band_count(side: int, n_angles: int, n_det: int, angles=None, factor: int = 1) -> float:
    """Ray-band visits of the level-`factor` forward (the bands whose left chord
    partner lies in [-1, n-1], as band_range in projector.cu), summed over all rays."""
    th = np.arange(n_angles) * (np.pi / n_angles)
    if angles is not None:
        th = th[np.asarray(angles)]
    c, s = np.cos(th), np.sin(th)
    c[np.abs(c) < 1e-14] = 0.0
    s[np.abs(s) < 1e-14] = 0.0
    h = float(factor)
    n, half, t0 = side // factor, side / 2.0, -(n_det - 1) / 2.0
    row = np.abs(c) >= np.abs(s)
    a_, b_ = np.where(row, c, s), np.where(row, s, c)  # band-normal / along-band cosines
    xi_dj = 1.0 / (a_ * h)
    xi_base = t0 / (a_ * h) + (half - h / 2) * b_ / (a_ * h) + half / h - 0.5
    step = -b_ / a_
    x0 = xi_base[:, None] + np.arange(n_det)[None, :] * xi_dj[:, None]
    st = np.broadcast_to(step[:, None], x0.shape)
    with np.errstate(divide="ignore", invalid="ignore"):
        e1 = (-1.0 - x0) / st
        e2 = (n - x0) / st
    lo = np.clip(np.ceil(np.minimum(e1, e2)), 0, n)
    hi = np.clip(np.ceil(np.maximum(e1, e2)), 0, n)
    cnt = np.where(st == 0, np.where((x0 >= -1) & (x0 < n), n, 0), np.maximum(hi - lo, 0))
    return float(cnt.sum())


def adjoint_window_reads(side: int, n_angles: int, factor: int) -> float:
    """Shared-memory bytes the level-`factor` adjoint reads: factor 1 one 16-byte
    element (two bins of a pixel and of its mirror) per pixel pair and angle, i.e.
    8 B per pixel-angle; coarser levels one 8-byte element (a bin of both mirror
    rows) per candidate bin (nb = floor(2R) + 1) per pixel pair and angle."""
    n = side // factor
    if factor == 1:
        return 8.0 * n * n * n_angles
    th = np.arange(n_angles) * (np.pi / n_angles)
    R = (np.abs(np.cos(th)) + np.abs(np.sin(th))) * factor / 2.0
    nb = np.floor(2 * R) + 1
    return 4.0 * n * n * float(nb.sum())


def projector_microbench(device, reps: int = 100, shard_reps: int = 20, smem_peak_gbs=None,
                         hbm_peak_gbs=None) -> dict:
    """Config E: forward K and adjoint K^T alone on the seeded
    2048^2 ellipse image (2048 angles x 2897 bins) at every level f = 1..64,
    median of `reps` CUDA-event timed launches each (L2 warm: a projector's
    operands are on-chip between launches anyway); per level the algorithmic
    HBM GB/s (4 (d_i + m) bytes per apply), the shared-memory bytes the kernels
    read against the live shared-memory peak, and the angle-sharded runs at
    2/4/8 ranks (every rank's shard plan timed alone on this GPU, max over
    ranks: compute only, no collective)."""
    import torch

    from paper_2412_10249_b200 import ctmodel, mrsketch
    from paper_2412_10249_b200.synth import CONFIGS, ellipse_phantom

    e = CONFIGS["E"]
    geom = ctmodel.Geometry(e.side, e.n_angles, e.n_det)
    x = torch.from_numpy(ellipse_phantom(e.side, 0).astype(np.float32)).to(device)
    y = torch.from_numpy(np.random.default_rng(7).standard_normal(geom.m).astype(np.float32)).to(device)
    stream = torch.cuda.current_stream(device)

    def med(fn, n_rep):
        for _ in range(3):
            fn()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(n_rep)]
        for a, b in ev:
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        return float(np.median([a.elapsed_time(b) for a, b in ev]))

    levels = [2 ** k for k in range(7)]
    us = {f: (x if f == 1 else mrsketch.decimate(x, f)).reshape(-1).contiguous() for f in levels}

    def time_plan(plan, ysl, n_rep):
        sino = torch.empty(plan.m_loc, device=device)
        res = {}
        for f in levels:
            bp = torch.empty(us[f].numel(), device=device)
            res[f] = (med(lambda: plan.project(us[f], f, sino), n_rep),
                      med(lambda: plan.backproject(ysl, f, bp), n_rep))
        return res

    one = time_plan(ctmodel.get_plan(geom), y, reps)
    out = {}
    for f in levels:
        fwd, adj = one[f]
        di = (e.side // f) ** 2
        hbm_bytes = 4.0 * (di + geom.m)
        nnz = 4.0 / np.pi * e.n_angles * e.side * e.side / f
        f_smem = 8.0 * ray_band_count(e.side, e.n_angles, e.n_det, factor=f)
        a_smem = adjoint_window_reads(e.side, e.n_angles, f)
        row = {"forward_ms": round(fwd, 4), "adjoint_ms": round(adj, 4),
               "fwd_adj_pairs_per_s": round(1e3 / (fwd + adj), 1),
               "footprint_evals_per_s": round(2 * nnz / ((fwd + adj) * 1e-3), 1),
               "hbm_bytes_per_apply": hbm_bytes,
               "forward_hbm_gbs": round(hbm_bytes / (fwd * 1e-3) / 1e9, 1),
               "adjoint_hbm_gbs": round(hbm_bytes / (adj * 1e-3) / 1e9, 1)}
        if hbm_peak_gbs:
            row["forward_hbm_frac"] = round(row["forward_hbm_gbs"] / hbm_peak_gbs, 5)
            row["adjoint_hbm_frac"] = round(row["adjoint_hbm_gbs"] / hbm_peak_gbs, 5)
        if smem_peak_gbs:
            row["forward_smem_frac"] = round(f_smem / (fwd * 1e-3) / 1e9 / smem_peak_gbs, 4)
            row["adjoint_smem_frac"] = round(a_smem / (adj * 1e-3) / 1e9 / smem_peak_gbs, 4)
        out[f"f{f}"] = row
    sharded = {}
    for W in (2, 4, 8):
        worst = {f: [0.0, 0.0] for f in levels}
        for rank in range(W):
            rows = ctmodel.shard_angles(e.n_angles, rank, W)
            plan = ctmodel.Plan(geom, angles=rows, device=device)
            ysl = y.reshape(e.n_angles, e.n_det)[list(rows)].reshape(-1).contiguous()
            for f, (fw, ad) in time_plan(plan, ysl, shard_reps).items():
                worst[f][0] = max(worst[f][0], fw)
                worst[f][1] = max(worst[f][1], ad)
            del plan
        sharded[f"world{W}"] = {
            f"f{f}": {"forward_ms_max_rank": round(fw, 4), "adjoint_ms_max_rank": round(ad, 4),
                      "efficiency": round((one[f][0] + one[f][1]) / (W * (fw + ad)), 3)}
            for f, (fw, ad) in worst.items()}
    return {"config": f"E: {e.side}^2, {e.n_angles} angles x {e.n_det} bins, levels f = 1..64",
            "reps": reps, "statistic": "median", "levels": out,
            "sharded": sharded,
            "sharded_note": f"each rank's mirror-closed shard plan timed alone on this GPU "
                            f"({shard_reps} reps, median), max over ranks; compute only (no "
                            "all-reduce); efficiency = T_1 / (W T_W) of forward + adjoint"}


def cpu_reference(cfg, steps: int, warmup: int, sample: int = CPU_SAMPLE_ANGLES):
    """Reference algorithm (scipy CSR, float64) on `sample` evenly spaced angles of cfg.

    Per-level times of the sampled projector applies and sinogram-side updates
    are scaled by n_angles/sample; the image-side update (full d) is timed as is.
    Returns (iters/s, details).
    """
    from oracle import sketch_oracle as sk
    from oracle import solver_oracle as so

    r = cfg.levels
    probs = [1.0 / r] * r
    sel = np.linspace(0, cfg.n_angles, sample, endpoint=False).astype(np.int64)
    t_build = time.perf_counter()
    ops = so.SketchedCT(cfg.side, cfg.n_angles, cfg.n_det, probs, angle_idx=sel)
    t_build = time.perf_counter() - t_build
    # every host core the process may use: the CSR matvecs (the reference's hot
    # loop) run as row blocks on a thread pool (scipy releases the GIL)
    from concurrent.futures import ThreadPoolExecutor

    threads = max(1, len(os.sched_getaffinity(0)))
    pool = ThreadPoolExecutor(threads)
    for p in ops.proj.values():
        p.set_threads(pool, threads)
    scale = cfg.n_angles / sample
    rng = np.random.default_rng(0)
    x = rng.random(cfg.d)
    y = rng.standard_normal(ops.m)
    b = rng.standard_normal(ops.m)
    tab = rng.standard_normal(ops.m)
    st = so.init_state(ops, seed=SEED)
    per_level, per_level_1 = [], []
    for i in range(r):
        f = ops.factors[i]
        proj = ops.proj[f]
        xl = sk.decimate(x.reshape(cfg.side, cfg.side), f).ravel()
        reps = 3 if f <= 2 else 5
        # pure CSR matvecs of the sampled rows (scale with the angle count)
        t = time.perf_counter()
        for _ in range(reps):
            proj.adjoint_apply(y)
            proj.apply(xl)
        t_proj = (time.perf_counter() - t) / reps
        # sinogram-side elementwise of sketch_step on the sampled rows (scales)
        t = time.perf_counter()
        for _ in range(reps):
            zeta = (tab - st.psi[i]) + st.psi_sum
            _ = st.psi_sum + probs[i] * (tab - st.psi[i])
            _ = ((st.y + SIGMA * zeta) - SIGMA * b) / (1.0 + SIGMA)
        t_sino = (time.perf_counter() - t) / reps
        # the whole reference step on the sample: includes restriction / compensation /
        # prolongation and the image-side update at full size, which do not scale
        t = time.perf_counter()
        for _ in range(2):
            st.k = 0
            phi_new = ops.adjoint_apply(i, st.y)
            psi_new = ops.apply(i, st.x)
            xi = (phi_new - st.phi[i]) + st.phi_sum
            zeta = (psi_new - st.psi[i]) + st.psi_sum
            st.phi_sum = st.phi_sum + probs[i] * (phi_new - st.phi[i])
            st.psi_sum = st.psi_sum + probs[i] * (psi_new - st.psi[i])
            st.phi[i] = phi_new
            st.psi[i] = psi_new
            st.x = (st.x - 1.0 * xi) / (1.0 + 1e-2)
            st.y = ((st.y + SIGMA * zeta) - SIGMA * b) / (1.0 + SIGMA)
        t_step = (time.perf_counter() - t) / 2
        t_img = max(t_step - t_proj - t_sino, 0.0)
        per_level.append(scale * (t_proj + t_sino) + t_img)
        # the same CSR matvecs on one core (the reference's own execution)
        proj.set_threads(pool, 1)
        t = time.perf_counter()
        for _ in range(reps):
            proj.adjoint_apply(y)
            proj.apply(xl)
        t_proj1 = (time.perf_counter() - t) / reps
        proj.set_threads(pool, threads)
        per_level_1.append(scale * (t_proj1 + t_sino) + t_img)
    sched = so.level_schedule(SEED, warmup, steps, probs)
    t_iter = float(np.mean([per_level[int(i)] for i in sched]))
    t_iter_1 = float(np.mean([per_level_1[int(i)] for i in sched]))
    detail = {
        "sample": f"{sample} of {cfg.n_angles} angles (every {cfg.n_angles // sample}th), all "
                  f"{r} levels; CSR matvec + sinogram-side time x{scale:g}, image-side work (restriction, "
                  f"compensation, prolongation, primal update; full size) as measured; "
                  f"mean over the timed steps' level schedule",
        "per_level_s": [round(v, 6) for v in per_level],
        "single_core_per_level_s": [round(v, 6) for v in per_level_1],
        "single_core_iters_per_s": 1.0 / t_iter_1,
        "extrapolated": True,
        "csr_build_s_excluded": round(t_build, 3),
        "threads": threads,
        "threading": "CSR matvecs split into row blocks over a thread pool; the numpy "
                     "elementwise image/sinogram-side work is single-threaded as in the reference",
    }
    pool.shutdown()
    return 1.0 / t_iter, detail


def cpu_reference_full(key: str = "C", steps: int = 8, warm: int = 2) -> dict:
    """The reference algorithm (oracle/ restatement: scipy CSR float64, the
    reference's sketch_step) on the FULL operator of config `key`, every step
    timed with perf_counter, nothing extrapolated: `steps` iterations of the
    seeded level schedule after `warm` untimed ones, with the CSR matvecs on
    every host core, then 3 iterations on one core. CSR build time is reported
    separately (the reference caches its matrices)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import solver_oracle as so
    from paper_2412_10249_b200.synth import CONFIGS

    cfg = CONFIGS[key]
    r = cfg.levels
    probs = [1.0 / r] * r
    t0 = time.perf_counter()
    ops = so.SketchedCT(cfg.side, cfg.n_angles, cfg.n_det, probs)
    build_s = time.perf_counter() - t0
    threads = max(1, len(os.sched_getaffinity(0)))
    pool = ThreadPoolExecutor(threads)
    rng = np.random.default_rng(1)
    b = rng.standard_normal(ops.m)
    st = so.init_state(ops, seed=SEED)
    sched = so.level_schedule(SEED, 0, warm + steps + 3, probs)

    def run(n_threads, ks):
        for p in ops.proj.values():
            p.set_threads(pool, n_threads)
        out = []
        for k in ks:
            t = time.perf_counter()
            so.sketch_step(st, ops, b, SIGMA, cfg.mu_g, cfg.mu_g)
            out.append(time.perf_counter() - t)
        return out

    run(threads, range(warm))
    times = run(threads, range(warm, warm + steps))
    times1 = run(1, range(warm + steps, warm + steps + 3))
    pool.shutdown()
    lev = [int(v) for v in sched[:warm + steps + 3]]
    return {"config": f"{cfg.name}: {cfg.side}^2, {cfg.n_angles} angles x {cfg.n_det} bins, "
                      f"r={r}, full operator (no sampling)",
            "iters_per_s": steps / sum(times), "threads": threads,
            "step_s": [round(v, 4) for v in times], "levels": lev[warm:warm + steps],
            "single_core_iters_per_s": 3 / sum(times1),
            "single_core_step_s": [round(v, 4) for v in times1],
            "single_core_levels": lev[warm + steps:],
            "csr_build_s_excluded": round(build_s, 1), "extrapolated": False}


def native_config_c(device, steps: int = 100, warmup: int = 10) -> dict:
    """The native step on config C (512^2 / 720 / 725, r = 5), timed as the
    headline (device events, L2 flushed between steps): the configuration the
    reference's fully timed solve (--impl reference, measured_full_operator) runs."""
    import torch

    from paper_2412_10249_b200 import dist as dist_mod
    from paper_2412_10249_b200 import ctmodel, mrsketch, solvers
    from paper_2412_10249_b200.synth import CONFIGS

    cfg = CONFIGS["C"]
    r = cfg.levels
    geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    b = np.random.default_rng(1).standard_normal(geom.m)
    fam = mrsketch.make_family(r, cfg.side, [1.0 / r] * r, mode="coarse")
    prob = dist_mod.make_sharded_problem(geom, b, fam, cfg.mu_g)
    eng = prob.engine
    st = solvers.init_state(prob, seed=SEED)
    prm = solvers._params(SIGMA, cfg.mu_g, cfg.mu_g)
    eng.capture_all(st, prm)
    for lv in range(r):
        for _ in range(2):
            solvers._device_step(eng, st, lv, prm)
    sched = solvers.draw_levels(SEED, 0, warmup + steps, prob.cum_probs)
    for k in range(warmup):
        solvers._device_step(eng, st, int(sched[k]), prm)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    stream = torch.cuda.current_stream(device)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    torch.cuda.synchronize()
    for k, (a, c) in enumerate(ev):
        flush.zero_()
        a.record(stream)
        solvers._device_step(eng, st, int(sched[warmup + k]), prm)
        c.record(stream)
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(c) for a, c in ev])
    return {"config": f"{cfg.name}: {cfg.side}^2, {cfg.n_angles} angles x {cfg.n_det} bins, r={r}",
            "value": steps / (ms.sum() / 1e3), "unit": "iter/s", "steps": steps,
            "l2": "flushed between steps"}


# ---------------------------------------------------------------- native arm

def clocks_sampler(path):
    try:
        return subprocess.Popen(
            ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
             "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
            stdout=open(path, "w"), stderr=subprocess.DEVNULL,
        )
    except Exception:
        return None


def summarize_clocks(path, dev_index):
    sm, smax, reasons = [], None, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    try:
        for line in open(path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9 or parts[0] != str(dev_index):
                continue
            sm.append(float(parts[1]))
            smax = float(parts[2])
            for name, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
    except Exception:
        pass
    return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
            "reasons": sorted(reasons), "samples": len(sm)}


def main():
    args = parse()
    from paper_2412_10249_b200.synth import CONFIGS

    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n_gpus = world  # the GPUs actually used (one process per GPU under torchrun)
    if args.gpus != world:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: launch N > 1 under "
              "torch.distributed.run; measuring {world} GPU(s)".replace("{world}", str(world)),
              file=sys.stderr)

    base = {
        "metric": "imask_iters_per_sec",
        "unit": "iter/s",
        "n_gpus": n_gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded 10-ellipse phantom, b = Kx + 1% gaussian noise)",
    }
    workload = {"workload": f"ImaSk sketch_step, config {cfg.name}: {cfg.side}^2 image, "
                            f"{cfg.n_angles} angles x {cfg.n_det} bins, r={cfg.levels} levels "
                            f"(factors 1..{2 ** (cfg.levels - 1)}), uniform level probabilities",
                "side": cfg.side, "n_angles": cfg.n_angles, "n_det": cfg.n_det,
                "levels": cfg.levels, "seed": SEED, "sigma": SIGMA, "mu_g": cfg.mu_g,
                "parallelism": (f"mirror-closed angle shards x{n_gpus}, NCCL all-reduce of the "
                                "coarse backprojection (one CUDA graph per step)"
                                if n_gpus > 1 or args.collective else "single GPU")}

    if args.impl == "reference":
        if world > 1 and rank != 0:
            return
        t0 = time.perf_counter()
        ips, det = cpu_reference(cfg, args.steps, args.warmup)
        cores = det["threads"]
        # the largest config whose full operator the reference's CSR route builds in
        # about a minute (and ~28 GB) is C; smaller configs time themselves
        full_key = args.config if args.config in ("A", "B", "C") else "C"
        full_c = None if args.no_full_reference else cpu_reference_full(full_key)
        line = dict(base, impl="reference", value=ips, ms_per_step=1e3 / ips,
                    extrapolated=True,
                    config=dict(workload, l2="n/a (CPU)"),
                    cpu_baseline={"value": ips, "unit": "iter/s", "cores": cores, "kind": "port",
                                  "sample": det["sample"], "extrapolated": True,
                                  "single_core_value": det.get("single_core_iters_per_s")},
                    e2e={"value": ips, "unit": "iter/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0},
                    measured_full_operator=full_c,
                    reference_detail=dict(det, wall_s=round(time.perf_counter() - t0, 2),
                                          timing_note=(
                                              "value and ms_per_step are the per-step time of the "
                                              "full config-D step modelled from timed sampled-angle "
                                              "steps (extrapolated: the full CSR needs ~130 GB and "
                                              "~5 min to build); measured_full_operator is a "
                                              "fully timed, non-extrapolated reference solve "
                                              "(config C for D)")))
        print(json.dumps(line))
        return

    import torch

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    group = None
    dist_on = world > 1 or args.collective
    if dist_on:
        import torch.distributed as dist

        if "MASTER_ADDR" not in os.environ:  # --collective without torchrun: a group of one
            import socket

            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0",
                              WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=device)
        group = dist.group.WORLD

    from paper_2412_10249_b200 import ctmodel, mrsketch, solvers
    from paper_2412_10249_b200 import dist as dist_mod
    from paper_2412_10249_b200.synth import ellipse_phantom

    r = cfg.levels
    probs = [1.0 / r] * r
    geom = ctmodel.Geometry(cfg.side, cfg.n_angles, cfg.n_det)
    x_true = ellipse_phantom(cfg.side, 0)
    # data: b = K x_true + 1% noise, built with the device projector (the CSR oracle needs
    # ~130 GB at this size); the same seeded arrays on every rank
    full_plan = ctmodel.get_plan(geom)
    sino = full_plan.project(torch.from_numpy(x_true.astype(np.float32).ravel()).to(device), 1)
    sino_h = sino.double().cpu().numpy()
    noise = np.random.default_rng(1).standard_normal(sino_h.size)
    b_full = sino_h + cfg.kappa * np.abs(sino_h).max() * noise
    b_loc = dist_mod.local_rows(geom, b_full, rank, world)  # mirror-closed shard rows

    fam = mrsketch.make_family(r, cfg.side, probs, mode="coarse")
    prob = dist_mod.make_sharded_problem(geom, b_loc, fam, cfg.mu_g, rank, world, group)
    eng = prob.engine
    st = solvers.init_state(prob, seed=SEED)
    prm = solvers._params(SIGMA, cfg.mu_g, cfg.mu_g)
    sched = solvers.draw_levels(SEED, 0, args.warmup + args.steps, prob.cum_probs)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # warm-up; the per-level CUDA graphs are captured (and uploaded) here, never inside
    # the timed region, and every one of them (each level at both dual-buffer
    # parities) is launched once before the W schedule steps
    eng.capture_all(st, prm)
    for lv in range(r):
        for _ in range(2):
            solvers._device_step(eng, st, lv, prm)
    for k in range(args.warmup):
        solvers._device_step(eng, st, int(sched[k]), prm)
    torch.cuda.synchronize()

    # timed: per-step events on the launching stream, L2 flushed between steps
    stream = torch.cuda.current_stream(device)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clk_path = os.path.join(REPO, f".clocks_rank{rank}.csv")
    sampler = clocks_sampler(clk_path) if rank == 0 else None
    time.sleep(0.3)
    launches = 0
    barrier()
    torch.cuda.synchronize()
    for s in range(args.steps):
        flush.zero_()
        starts[s].record(stream)
        launches += solvers._device_step(eng, st, int(sched[args.warmup + s]), prm)
        ends[s].record(stream)
    torch.cuda.synchronize()
    barrier()
    if sampler:
        sampler.terminate()
        sampler.wait()
    step_ms = np.array([a.elapsed_time(b) for a, b in zip(starts, ends)])
    total_ms = float(step_ms.sum())
    if world > 1:
        t = torch.tensor([total_ms], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ips = args.steps / (total_ms / 1e3)
    level_counts = np.bincount(sched[args.warmup:], minlength=r).tolist()
    lev = np.asarray(sched[args.warmup:])
    per_level_ms = {f"f{2 ** (r - 1 - i)}": round(float(step_ms[lev == i].mean()), 4)
                    for i in range(r) if np.any(lev == i)}
    # the sampled schedule's level mix varies with K; the uniform-probability
    # expectation over the same per-level means does not
    uniform_ips = (1e3 / float(np.mean(list(per_level_ms.values())))
                   if len(per_level_ms) == r else None)

    if args.steps_only:
        if rank == 0:
            print(json.dumps(dict(base, value=ips, ms_per_step=total_ms / args.steps,
                                  gpu_launches=launches, per_level_ms=per_level_ms,
                                  note="--steps-only: no roofline / e2e / cpu_baseline")))
        if dist_on:
            torch.distributed.destroy_process_group()
        return

    # dominant kernel: level-1 (f = 1) projector, timed alone with events
    plan = eng.plan
    ybuf = st.y.clone()
    out = torch.empty(cfg.d, device=device)
    reps = 20
    for _ in range(3):
        plan.backproject(ybuf, 1, out)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for q in range(reps):
        flush.zero_()
        ev[2 * q].record(stream)
        plan.backproject(ybuf, 1, out)
        ev[2 * q + 1].record(stream)
    torch.cuda.synchronize()
    adj_ms = float(np.mean([ev[2 * q].elapsed_time(ev[2 * q + 1]) for q in range(reps)]))
    for q in range(reps):
        flush.zero_()
        ev[2 * q].record(stream)
        plan.project(st.x, 1, ybuf)
        ev[2 * q + 1].record(stream)
    torch.cuda.synchronize()
    fwd_ms = float(np.mean([ev[2 * q].elapsed_time(ev[2 * q + 1]) for q in range(reps)]))
    n_loc = len(ctmodel.shard_angles(cfg.n_angles, rank, world))
    m_loc = n_loc * cfg.n_det
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    traffic_tab = {}
    try:
        traffic_tab = json.load(open(os.path.join(REPO, "profiles", "traffic.json")))
    except Exception:
        pass

    # HBM-bound kernels (SURVEY 8(d) kernel (3)+(4)): the image-side SAGA update
    # with the fused compensation pyramid, timed alone at the full and coarsest level
    import ctypes
    from paper_2412_10249_b200 import _lib

    cst = st.c_state(eng.b)
    flush_sink = torch.empty((), device=device)

    def time_image(level0):
        for _ in range(3):
            _lib.check(_lib.lib().imask_step_image(plan.handle, ctypes.byref(cst), level0,
                                                   ctypes.byref(prm), plan.stream))
        for q in range(reps):
            # read-flush: evicts the working set without leaving dirty lines whose
            # write-back would be charged to the kernel under test
            flush_sink.copy_(flush.sum())
            ev[2 * q].record(stream)
            _lib.check(_lib.lib().imask_step_image(plan.handle, ctypes.byref(cst), level0,
                                                   ctypes.byref(prm), plan.stream))
            ev[2 * q + 1].record(stream)
        torch.cuda.synchronize()
        return float(np.mean([ev[2 * q].elapsed_time(ev[2 * q + 1]) for q in range(reps)]))

    # the same launch back to back over rotating image-side buffer sets (x, phi_sum,
    # phi table, bp) whose total exceeds L2, events around the whole batch: the
    # per-launch time without the ~6 us an event pair adds around one small launch
    # (tools/probes/stream_probe.cu: an empty kernel reads 6.1 us between events,
    # a plain float4 kernel of the same traffic 8.2 / 10.2 us cold and 6.3 / 7.8 us
    # back to back, whatever its grid shape)
    n_sets = 12
    tab_len = st.phi_tab.numel()
    sets = []
    for _ in range(n_sets):
        bufs = [torch.zeros(cfg.d, device=device) for _ in range(3)] + \
               [torch.zeros(tab_len, device=device)]
        cs = _lib.ImaskState(bufs[0].data_ptr(), st.y.data_ptr(), eng.b.data_ptr(),
                             bufs[1].data_ptr(), st.psi_sum.data_ptr(), bufs[3].data_ptr(),
                             st.psi_tab.data_ptr(), bufs[2].data_ptr(), None, None)
        sets.append((bufs, cs))

    def time_image_b2b(level0):
        rounds = []
        for q in range(8):
            flush_sink.copy_(flush.sum())
            ev[0].record(stream)
            for _, cs in sets:
                _lib.check(_lib.lib().imask_step_image(plan.handle, ctypes.byref(cs), level0,
                                                       ctypes.byref(prm), plan.stream))
            ev[1].record(stream)
            torch.cuda.synchronize()
            if q >= 2:
                rounds.append(ev[0].elapsed_time(ev[1]) / n_sets)
        return float(np.median(rounds))

    hbm_kernels = []
    for level0, name in ((r - 1, "k_saga_image_full32 (f=1, compensation fused)"),
                         (0, f"k_saga_image_coarse32 (f={2 ** (r - 1)})")):
        f = 2 ** (r - 1 - level0)
        di = cfg.d // (f * f)
        nbytes = 4.0 * (7 * cfg.d) if f == 1 else 4.0 * (4 * cfg.d + 3 * di)
        ms = time_image(level0)
        gbs = nbytes / (ms * 1e-3) / 1e9
        ms_b = time_image_b2b(level0)
        gbs_b = nbytes / (ms_b * 1e-3) / 1e9
        hbm_kernels.append({"kernel": name, "algorithmic_bytes": nbytes, "avg_launch_ms": round(ms, 4),
                            "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                            "frac": round(gbs / hbm_peak, 4),
                            "back_to_back": {
                                "avg_launch_ms": round(ms_b, 4), "achieved": round(gbs_b, 1),
                                "frac": round(gbs_b / hbm_peak, 4), "sets": n_sets,
                                "note": "launches over rotating buffer sets larger than L2, "
                                        "events around the batch (no per-launch event overhead)"},
                            "traffic": traffic_tab.get("saga_image_full" if f == 1 else
                                                       "saga_image_coarse"),
                            "traffic_note": "ncu DRAM bytes of the launch inside the fused step "
                                            "(profiles/traffic.json), which reads the adjoint's "
                                            "split planes (4 B x planes x n^2, L2-resident in the "
                                            "real step, cold under ncu) in place of bp; the timed "
                                            "launch here reads bp"})

    # dominant kernel of the step: the level-1 projector (forward or adjoint, whichever
    # is slower). It is FP32-issue bound; the HBM figure uses its compulsory
    # bytes 4*(d + m_slab) and is small by construction; fp32_view carries the real bound.
    fwd_dominant = fwd_ms >= adj_ms
    dom_ms = fwd_ms if fwd_dominant else adj_ms
    alg_bytes = 4.0 * (cfg.d + m_loc)
    achieved = alg_bytes / (dom_ms * 1e-3) / 1e9
    nnz = 4.0 / np.pi * n_loc * cfg.d  # footprint evaluations = nnz of the reference CSR
    ffma = ctypes.c_double(0.0)
    _lib.check(_lib.lib().imask_probe_ffma_peak(local, ctypes.byref(ffma)))
    smem = ctypes.c_double(0.0)
    _lib.check(_lib.lib().imask_probe_smem_peak(local, ctypes.byref(smem)))
    smem_peak = smem.value / 1e9
    # shared-memory bytes the kernels must read: the forward one 8-byte value
    # pair and one difference pair per band for a ray and its mirror (8 B per
    # ray-band); the adjoint one 16-byte window element per pixel and angle pair
    # (8 B per pixel-angle)
    shard = ctmodel.shard_angles(cfg.n_angles, rank, world)
    fwd_smem = 8.0 * ray_band_count(cfg.side, cfg.n_angles, cfg.n_det, shard)
    adj_smem = 8.0 * cfg.d * n_loc
    smem_view = {
        "peak": round(smem_peak, 1), "unit": "GB/s",
        "peak_source": "live probe (imask_probe_smem_peak: conflict-free LDS.128 on every SM)",
        "forward_f1": {"bytes": fwd_smem, "achieved": round(fwd_smem / (fwd_ms * 1e-3) / 1e9, 1),
                       "frac": round(fwd_smem / (fwd_ms * 1e-3) / 1e9 / smem_peak, 4)},
        "adjoint_f1": {"bytes": adj_smem, "achieved": round(adj_smem / (adj_ms * 1e-3) / 1e9, 1),
                       "frac": round(adj_smem / (adj_ms * 1e-3) / 1e9 / smem_peak, 4)}}
    roofline = {"bound": "hbm",
                "kernel": ("k_forward_tma<false> (level-1 projection)" if fwd_dominant
                           else "k_adjoint<pair,sym> (level-1 backprojection)"),
                "achieved": round(achieved, 2), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 5),
                "traffic": traffic_tab.get("forward_f1" if fwd_dominant else "adjoint_f1"),
                "algorithmic_bytes": alg_bytes, "avg_launch_ms": round(dom_ms, 4),
                "peak_source": peak_src,
                "note": "projectors are bound by shared-memory bandwidth and instruction issue, "
                        "not HBM (SURVEY 8(d)): see smem_view and fp32_view; HBM-bound kernels "
                        "in hbm_kernels",
                "fp32_view": {
                    "footprint_evals": nnz,
                    "forward_f1_ms": round(fwd_ms, 4), "adjoint_f1_ms": round(adj_ms, 4),
                    "forward_evals_per_s": round(nnz / (fwd_ms * 1e-3), 1),
                    "adjoint_evals_per_s": round(nnz / (adj_ms * 1e-3), 1),
                    "ffma_peak_per_s": round(ffma.value, 1),
                    "evals_per_ffma_slot": round(nnz / (dom_ms * 1e-3) / ffma.value, 4),
                    "csr_equivalent_gbs": round(8.0 * nnz / (dom_ms * 1e-3) / 1e9, 1),
                    "csr_note": "bandwidth a float32 value + int32 index CSR SpMV would need "
                                "to match this kernel (the reference's operator form)"},
                "smem_view": smem_view,
                "hbm_kernels": hbm_kernels}

    # e2e through the public API: solvers.run with host inputs (every rank runs its
    # shard under torchrun; the job time is the max over ranks)
    e2e = None
    if not args.no_e2e:
        e2e_steps = min(args.steps, 200)
        b_host = torch.from_numpy(b_loc.astype(np.float32)).pin_memory()
        xref_host = torch.from_numpy(x_true.astype(np.float32).ravel()).pin_memory()
        # untimed warm-up of the same call: first-use module loads of the metric path
        # and the step graphs of every level (cached with the plan, re-targeted to
        # the timed run's buffers if they differ)
        prob_w = dist_mod.make_sharded_problem(geom, b_host.to(device), fam, cfg.mu_g,
                                               rank, world, group)
        prob_w.engine.capture_all(solvers.init_state(prob_w, seed=SEED), prm)
        x_out = torch.empty(cfg.d, dtype=torch.float32).pin_memory()
        rep_w = solvers.run(prob_w, "sketch", SIGMA, cfg.mu_g, e2e_steps, record_every=1,
                            seed=SEED, x_ref=xref_host.to(device))
        x_out.copy_(rep_w.x)  # the warm-up is the identical call, read-back included
        del prob_w, rep_w
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        b_dev = b_host.to(device, non_blocking=True)
        xref_dev = xref_host.to(device, non_blocking=True)
        prob2 = dist_mod.make_sharded_problem(geom, b_dev, fam, cfg.mu_g, rank, world, group)
        t1 = time.perf_counter()
        rep = solvers.run(prob2, "sketch", SIGMA, cfg.mu_g, e2e_steps, record_every=1,
                          seed=SEED, x_ref=xref_dev)
        t2 = time.perf_counter()
        x_out.copy_(rep.x)  # final iterate to pinned host memory
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        if rank == 0:
            print(f"[bench] e2e: setup {1e3 * (t1 - t0):.1f} ms, run {1e3 * (t2 - t1):.1f} ms, "
                  f"read-back {1e3 * (time.perf_counter() - t2):.1f} ms, step-graph re-targets "
                  f"{prob2.engine.graph_updates}", file=sys.stderr)
        e2e = {"value": e2e_steps / dt, "unit": "iter/s",
               "h2d_bytes_per_step": round((b_host.numel() + xref_host.numel()) * 4 / e2e_steps),
               "d2h_bytes_per_step": round(8 + x_out.numel() * 4 / e2e_steps),
               "api": "solvers.run(prob, 'sketch', ..., record_every=1, x_ref=...)",
               "steps": e2e_steps,
               "timing": "host wall clock around the call, max over ranks"}

    micro = None
    if not args.no_microbench and world == 1:
        micro = projector_microbench(device, smem_peak_gbs=smem_peak, hbm_peak_gbs=hbm_peak)
    config_c = native_config_c(device) if (world == 1 and not args.no_microbench) else None

    cpu = None
    if not args.no_cpu_baseline and rank == 0:
        cps, det = cpu_reference(cfg, args.steps, args.warmup)
        cpu = {"value": cps, "unit": "iter/s", "cores": det["threads"], "kind": "port",
               "sample": det["sample"], "per_level_s": det["per_level_s"], "extrapolated": True,
               "single_core_value": det["single_core_iters_per_s"]}

    clocks = summarize_clocks(clk_path, local) if rank == 0 else None
    if rank == 0:
        line = dict(base, value=ips, ms_per_step=total_ms / args.steps,
                    config=dict(workload, l2="flushed between steps (256 MiB write outside the "
                                             "per-step CUDA events)"),
                    e2e=e2e, roofline=roofline, cpu_baseline=cpu, clocks=clocks,
                    projector_microbench=micro,
                    gpu_launches=launches, per_level_ms=per_level_ms, level_counts=level_counts,
                    uniform_expectation={
                        "value": uniform_ips, "unit": "iter/s",
                        "note": "1 / (mean of per_level_ms over the r levels): the expected rate "
                                "under the uniform level probabilities, independent of how often "
                                "this K-step schedule drew each level"},
                    config_C=config_c)
        print(json.dumps(line))
        try:
            os.remove(clk_path)
        except OSError:
            pass
    if dist_on:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
