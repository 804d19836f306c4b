import os, subprocess, sys
import numpy as np
REPO = os.getcwd()
for g in [(128, 180, 183, 1), (256, 360, 363, 1), (1024, 1440, 1449, 1), (256, 360, 363, 2)]:
    outs = {}
    for name, extra in (("tma", {}), ("pair", {"IMASK_NO_QUAD": "1"}), ("l1", {"IMASK_NO_TMA": "1"})):
        env = dict(os.environ, OUT=f"/tmp/{name}.npy", **extra)
        r = subprocess.run([sys.executable, "tools/repro_quad.py", *map(str, g)], env=env, capture_output=True, text=True)
        if r.returncode: print(r.stderr[-2000:])
        outs[name] = np.load(f"/tmp/{name}.npy").reshape(g[1], g[2])
    for name in ("tma", "pair"):
        d = np.abs(outs[name] - outs["l1"]).sum(1)
        bad = np.nonzero(d > 1e-6 * np.abs(outs["l1"]).sum(1).max())[0]
        rel = np.linalg.norm(outs[name] - outs["l1"]) / np.linalg.norm(outs["l1"])
        print(g, name, "rel", rel, "bad rows", len(bad), bad[:20], flush=True)
