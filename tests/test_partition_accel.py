"""partition_accel against the reference partitioner: identical partition
trees (partitioner.tree_to_json) and lowered plans (plan.to_json), byte for
byte, over the reference's circuit families and the bench workloads.

Needs the reference package (importable in the build container only); the
GPU box has no copy, so the test skips there."""

import sys
import time
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")
if not REF.exists():
    pytest.skip("reference package not present", allow_module_level=True)
sys.path.insert(0, str(REF))

from svpart import circuits, qasm  # noqa: E402
from svpart import partitioner as P  # noqa: E402
from svpart import plan as ref_plan  # noqa: E402
from svpart.graph import build_graph  # noqa: E402

from paper_2509_14098_b200 import partition_accel, workloads  # noqa: E402

CASES = [(f"{fam}-{d}", lambda fam=fam, d=d: circuits.generate(fam, d, seed=3), h)
         for fam in ("ghz", "dj", "qft", "qpe", "ising", "su2random", "vqc")
         for d, h in ((8, [6, 3]), (12, [10, 6, 3]))]
CASES += [
    ("qft30", lambda: workloads.qft(30), [30, 12]),
    ("qv20", lambda: workloads.quantum_volume(20, seed=20), [18, 12]),
    ("qaoa24", lambda: workloads.qaoa_maxcut(24, seed=1), [22, 12]),
    ("sup24", lambda: workloads.random_supremacy(24, seed=2), [21, 12]),
]


def _run(src, budgets):
    g = build_graph(qasm.parse(src))
    t0 = time.perf_counter()
    tree = P.partition(g, P.make_hierarchy(budgets))
    dt = time.perf_counter() - t0
    return P.tree_to_json(tree), ref_plan.to_json(ref_plan.lower(tree)), dt


@pytest.mark.parametrize("name,make,budgets", CASES, ids=[c[0] for c in CASES])
def test_identical_trees_and_plans(name, make, budgets):
    src = make()
    partition_accel.uninstall()
    want_tree, want_plan, t_ref = _run(src, budgets)
    partition_accel.install()
    try:
        got_tree, got_plan, t_fast = _run(src, budgets)
    finally:
        partition_accel.uninstall()
    assert got_tree == want_tree
    assert got_plan == want_plan


def test_lazy_reach_matches_reference():
    """table.reach is still the reference's compute_reach when read."""
    from svpart.centrality import closeness as ref_closeness

    g = build_graph(qasm.parse(circuits.generate("qft", 6, seed=0)))
    fast, ref = partition_accel.closeness(g), ref_closeness(g)
    assert fast.cc == ref.cc and fast.n == ref.n
    assert dict(fast.reach) == ref.reach
