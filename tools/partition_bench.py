"""Reference partitioner vs partition_accel on the bench workloads: wall time
and byte-identical trees (needs the reference package, build container only).

    python tools/partition_bench.py
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

from svpart import partitioner as P, qasm  # noqa: E402
from svpart.graph import build_graph  # noqa: E402

from paper_2509_14098_b200 import partition_accel, workloads  # noqa: E402

for name, make, budgets in [
    ("QV-30 [30,12]", lambda: workloads.quantum_volume(30, seed=34), [30, 12]),
    ("QV-34 [33,12]", lambda: workloads.quantum_volume(34, seed=34), [33, 12]),
    ("QFT-34 [33,12]", lambda: workloads.qft(34), [33, 12]),
    ("QAOA-35 [32,12]", lambda: workloads.qaoa_maxcut(35, seed=35), [32, 12]),
]:
    g = build_graph(qasm.parse(make()))
    out = {}
    for mode in ("reference", "accel"):
        (partition_accel.install if mode == "accel" else partition_accel.uninstall)()
        t0 = time.perf_counter()
        tree = P.partition(g, P.make_hierarchy(budgets))
        out[mode] = (time.perf_counter() - t0, P.tree_to_json(tree))
    partition_accel.uninstall()
    (tr, jr), (ta, ja) = out["reference"], out["accel"]
    print(f"{name:16s} reference {tr:7.2f} s   accel {ta:6.2f} s   x{tr / ta:5.1f}   identical: {jr == ja}",
          flush=True)
