"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel name."""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki][:60]
    val = float(r[vi].replace(",", ""))
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + val)
unit = "us" if any(float(r[vi].replace(",", "")) > 1000 for r in rows[1:] if r[mi] == "gpu__time_duration.sum") else "?"
tot = sum(t for _, t in agg.values())
for k, (n, t) in agg.items():
    print(f"{k:60s} launches={n:3d} mean={t / n / 1e3:10.3f} us-share={100 * t / tot:5.1f}%")
