"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel.
usage: python tools/launch_shares.py [gpurun_out/launches.csv]"""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0, []])
for r in data:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    name = r[ki].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += v
    agg[name][2].append(v)
tot = sum(a[1] for a in agg.values())
for k, (n, t, vs) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.3f} ms {100 * t / tot:6.2f}%  n={n:3d}  per-launch min {min(vs):8.3f} ms  {k}")
