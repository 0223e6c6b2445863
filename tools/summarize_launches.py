"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
rows = []
with open(path) as f:
    lines = [l for l in f if not l.startswith("==")]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
    rows.append((r["Kernel Name"], v * scale))
agg = defaultdict(lambda: [0, 0.0])
for name, us in rows:
    key = name.split("(")[0][:90]
    agg[key][0] += 1
    agg[key][1] += us
total = sum(v[1] for v in agg.values())
print(f"{len(rows)} launches, {total:.1f} us total")
for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{us:10.1f} us {100*us/total:5.1f}%  x{c:5d}  avg {us/c:8.2f} us  {k}")
