"""Pin the CPU oracle against the reference's own outputs (tests/golden/, made by make_golden.py)."""

import numpy as np
import pytest

from conftest import plan_from_doc
from oracle import oracle as orc

TOL = 1e-12


@pytest.fixture(scope="module")
def backends():
    out = ["numpy", "c"]
    try:
        orc.kernels("ref")
        out.append("ref")
    except orc.OracleError:
        pass
    return out


def test_oracle_matches_reference_grid(grid_docs, grid_states, backends):
    n = 0
    for doc in grid_docs:
        if doc["name"] not in grid_states:
            continue
        plan = plan_from_doc(doc["plan"])
        backend = backends[n % len(backends)]
        blocks, st = orc.run_plan(plan, backend=backend)
        assert np.max(np.abs(blocks - grid_states[doc["name"]])) < TOL, (doc["name"], backend)
        assert st["task_counts"] == doc["stats"]["task_counts"]
        assert st["exchanges"] == doc["stats"]["exchanges"]
        dense = orc.gather(blocks, plan.layout_phases[-1], plan.d)
        assert np.max(np.abs(dense - grid_states[doc["name"] + "::dense"])) < TOL
        n += 1
    assert n >= 400


def test_oracle_cfg1_fingerprint(cfg1_docs, cfg1_fp):
    for key in ("18", "18_12"):
        plan = plan_from_doc(cfg1_docs[key]["plan"])
        blocks, _ = orc.run_plan(plan, backend="c", nthreads=4)
        flat = blocks.reshape(-1)
        assert np.max(np.abs(flat[cfg1_fp[key + "::idx"]] - cfg1_fp[key + "::amps"])) < 1e-12
        assert abs(flat.sum() - cfg1_fp[key + "::sum"][0]) < 1e-9


def test_oracle_rejects_protocol_errors(grid_docs):
    from paper_2509_14098_b200.plan import ExecutionPlan, Task

    doc = next(d for d in grid_docs if d["name"] == "ghz3-2")
    plan = plan_from_doc(doc["plan"])
    tasks = list(plan.tasks)
    tasks[1], tasks[5] = tasks[5], tasks[1]
    bad = ExecutionPlan(plan.d, plan.g, plan.layout_phases, tasks)
    with pytest.raises(orc.PlanInvalid):
        orc.run_plan(bad, backend="numpy")


def plan_ops(doc):
    """Gates in execution order, from the plan's ApplyFused payloads (a topological order)."""
    ops = []
    for t in doc["plan"]["tasks"]:
        if t["kind"] == "ApplyFused":
            ops += [(g["kind"], g["params"], g["qubits"]) for g in t["payload"]["gates"]]
    return ops


def test_dense_simulate_matches_reference(grid_docs, grid_states):
    # second dense route (executor.py:346-358) against the reference's gathered state
    n = 0
    for doc in grid_docs:
        if doc["name"] + "::dense" not in grid_states or doc["plan"]["d"] > 8:
            continue
        ref = orc.dense_simulate(doc["plan"]["d"], plan_ops(doc))
        assert orc.compare(ref, grid_states[doc["name"] + "::dense"]) < 1e-10, doc["name"]
        n += 1
    assert n > 100


@pytest.mark.parametrize("name", ["qaoa20_h18-12", "sup20_h19-12", "qft20_h19-12_x"])
def test_oracle_family_fingerprints(family_docs, family_fp, name):
    """The oracle on benchmark-family plans at 20 qubits against the reference's fingerprints."""
    from conftest import check_fingerprint, family_initial

    doc = family_docs[name]
    plan = plan_from_doc(doc["plan"])
    blocks, st = orc.run_plan(plan, backend="c", nthreads=4, initial=family_initial(doc))
    assert st["task_counts"] == doc["stats"]["task_counts"]
    assert st["exchanges"] == doc["stats"]["exchanges"]
    check_fingerprint(blocks.reshape(-1), family_fp, name, doc["fp_seed"], tol=1e-12)
