"""Per-launch table from an ncu launch-list CSV with gpu__time_duration.sum,
dram__bytes_read.sum and dram__bytes_write.sum (profiles/ summaries).

    python tools/launch_table.py gpurun_out/launches.csv "title" > profiles/x.txt
"""
import csv
import sys


def main(path: str, title: str) -> None:
    rows = list(csv.reader(line for line in open(path) if not line.startswith("==")))
    hdr = None
    by = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = (int(d["ID"]), d["Kernel Name"][:40])
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                     "Gbyte": 1e9}.get(d.get("Metric Unit", ""), 1.0)
            by.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * scale
    print(f"# {title}")
    print(f"# {path}: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
          "--clock-control none (cold-cache, serialised launches)")
    print(f"{'id':>4} {'kernel':40} {'us':>10} {'read GB':>9} {'write GB':>9} {'GB/s':>8}")
    for (i, k), m in sorted(by.items()):
        t = m.get("gpu__time_duration.sum", 0.0)
        rd = m.get("dram__bytes_read.sum", 0.0)
        wr = m.get("dram__bytes_write.sum", 0.0)
        print(f"{i:>4} {k:40} {t:10.1f} {rd / 1e9:9.4f} {wr / 1e9:9.4f} {(rd + wr) / max(t, 1e-9) / 1e3:8.0f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
