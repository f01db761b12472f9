"""GPU parity on the benchmark families at real tile geometry (D > K = 12).

The plans are QV / QAOA / supremacy / QFT circuits at 20-22 qubits on 1-4
ranks: every sweep then has fixed tile bits, so fixed-bit predicates,
per-tile slot tables, multi-row devices, sparse |0...0>-start sweeps and
the initial= load path run exactly as at 30+ qubits.  Each result is checked
against the reference's own fingerprint (tests/golden/make_golden.py
--families ran svpart.run_plan) and, amplitude by amplitude, against the
CPU oracle (oracle/sv_oracle.c on all host cores).
"""

import os

import numpy as np
import pytest

from conftest import check_fingerprint, family_initial, plan_from_doc

pytestmark = pytest.mark.gpu

TOL = 1e-10  # north_star: max-abs error 1e-10
NAMES = ["qv20_h18-12", "qv22_h22-12", "qv21_h20-12", "qaoa20_h18-12", "sup20_h19-12",
         "qft20_h19-12_x", "qv20_h20-12_x"]


@pytest.mark.parametrize("name", NAMES)
def test_family_matches_reference(family_docs, family_fp, name):
    from oracle import oracle as orc
    from paper_2509_14098_b200 import run_plan

    doc = family_docs[name]
    plan = plan_from_doc(doc["plan"])
    initial = family_initial(doc)
    res = run_plan(plan, initial=initial)
    assert res.stats.task_counts == doc["stats"]["task_counts"]
    assert res.stats.exchanges == doc["stats"]["exchanges"]
    assert res.state.phase == len(plan.layout_phases) - 1
    got = res.state.blocks.cpu().numpy()
    err = check_fingerprint(got.reshape(-1), family_fp, name, doc["fp_seed"], TOL)
    ref, _ = orc.run_plan(plan, backend="c", nthreads=os.cpu_count() or 1, initial=initial)
    full = float(np.max(np.abs(got - ref)))
    assert full < TOL, (name, full)
    print(f"{name}: fingerprint {err:.1e}, all {got.size} amplitudes vs oracle {full:.1e}")


def test_family_sparse_and_dense_starts_agree(family_docs):
    """The sparse |0...0> start (support-only sweeps) and full dense passes
    give bit-identical blocks: zero-filled loads and skipped zero tiles add
    only exact zeros."""
    from paper_2509_14098_b200 import executor, run_plan

    for name in ("qv20_h18-12", "sup20_h19-12"):
        plan = plan_from_doc(family_docs[name]["plan"])
        a = run_plan(plan).state.blocks.cpu().numpy()
        executor.SPARSE_START = False
        try:
            b = run_plan(plan).state.blocks.cpu().numpy()
        finally:
            executor.SPARSE_START = True
        assert np.array_equal(a, b), name
