"""Name of the slowest kernel launch in an ncu launch-list CSV (gpu__time_duration.sum)."""
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("=="))
        if r.get("Metric Name") == "gpu__time_duration.sum"]
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
best = max(rows, key=lambda r: float(r["Metric Value"].replace(",", "")) * scale.get(r.get("Metric Unit", ""), 1))
print(best["Kernel Name"].split("(")[0])
