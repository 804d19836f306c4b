"""The bench.py JSON contract (driver-facing): the reference arm on CPU, its
multi-rank behaviour, the multi-core CSR baseline, and (GPU) the native line's
keys on a small config."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def run_bench(args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    res = subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args,
                         capture_output=True, text=True, timeout=timeout, cwd=REPO, env=e)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    return [json.loads(ln) for ln in lines]


def test_reference_arm_line():
    (line,) = run_bench(["--impl", "reference", "--config", "A", "--steps", "3", "--warmup", "1"])
    assert BASE_KEYS <= set(line)
    assert line["impl"] == "reference" and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"],
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("ImaSk sketch_step")


def test_reference_arm_other_ranks_print_nothing():
    out = run_bench(["--impl", "reference", "--config", "A", "--steps", "2", "--warmup", "1"],
                    env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert out == []


def test_threaded_csr_equals_one_core():
    from concurrent.futures import ThreadPoolExecutor

    from oracle import ct_oracle

    op = ct_oracle.ProjectorOracle(64, 90, 91, 1)
    a, _ = op.csr_pair()
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal(op.domain_dim), rng.standard_normal(op.range_dim)
    fx, fy = op.apply(x), op.adjoint_apply(y)
    with ThreadPoolExecutor(4) as pool:
        op.set_threads(pool, 4)
        assert len(op._blocks[0]) > 1 and len(op._blocks[1]) > 1
        assert np.array_equal(op.apply(x), fx)
        assert np.array_equal(op.adjoint_apply(y), fy)


@pytest.mark.gpu
def test_native_line_keys():
    (line,) = run_bench(["--config", "A", "--steps", "6", "--warmup", "3", "--no-cpu-baseline",
                         "--no-microbench"])
    assert BASE_KEYS <= set(line)
    assert line["value"] > 0 and line["gpu_launches"] > 0
    rf = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf
    assert rf["bound"] in ("hbm", "tensor")
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
