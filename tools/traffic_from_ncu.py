"""Write profiles/traffic.json (per-launch DRAM bytes of the kernels bench.py
reports) from an ncu --set full report of tools/prof_step.py.

    python tools/traffic_from_ncu.py gpurun_out/prof_step.ncu-rep > profiles/traffic.json
"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
name_i, grid_i = hdr.index("Kernel Name"), hdr.index("launch__grid_size")
rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
units = rows[1]


def nbytes(r, i):
    v = float(r[i] or 0)
    u = units[i]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


launches = [(r[name_i], int(float(r[grid_i])), nbytes(r, rd) + nbytes(r, wr)) for r in rows[2:]]
res = {}
fwd = [b for n, g, b in launches if "k_forward_tma" in n]
# prof_step: imask_project for b (no SAGA), then steps at f=1, f=2, f=32
if fwd:
    # (the first launch of a level's TMA forward builds its chunk tables and reads
    # no image: the projection that builds b is the first launch with real traffic)
    real = [b for b in fwd if b > 1e6]
    res["forward_f1"] = int(real[0] if real else fwd[0])
adj = [b for n, g, b in launches if "k_adjoint<1, 32, 1" in n]
if adj:
    res["adjoint_f1"] = int(adj[0])
full = [b for n, g, b in launches if "k_saga_image_full" in n]
if full:
    res["saga_image_full"] = int(full[0])
coarse = [b for n, g, b in launches if "k_saga_image_coarse" in n]
if coarse:
    res["saga_image_coarse"] = int(coarse[-1])
res["_source"] = ("ncu --set full of tools/prof_step.py (imask_project for b, then one eager "
                  "sketch_step at f=1, f=2, f=32); dram__bytes_read.sum + dram__bytes_write.sum "
                  "per launch; saga_image_coarse is the f=32 launch")
print(json.dumps(res, indent=1))
