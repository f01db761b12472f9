"""Summarise an ncu launch-list CSV (gpu__time_duration.sum) per kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
per = defaultdict(list)
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1.0)
        per[r["Kernel Name"][:60]].append(v * scale)
tot = sum(sum(v) for v in per.values())
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):10.3f} ms {100*sum(v)/tot:5.1f}%  n={len(v):4d}  {k}  " + " ".join(f"{x:.2f}" for x in v[:12]))
