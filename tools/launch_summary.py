"""Summarise an ncu --csv launch list (gpu__time_duration) per kernel and grid."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[(r[ki].split("(")[0].replace("void ", "")[:44], r[gi])].append(float(r[vi]))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[0]:46s} {k[1]:14s} n={len(v):3d} mean={sum(v)/len(v)/1000:9.1f}us share={sum(v)/tot:6.1%}")
