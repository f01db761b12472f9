"""GPU parity: the CUDA executor against the reference's golden outputs and the oracle."""

import numpy as np
import pytest

from conftest import plan_from_doc

pytestmark = pytest.mark.gpu

TOL = 1e-10  # north_star: max-abs error 1e-10


def _run(plan, **kw):
    from paper_2509_14098_b200 import run_plan

    return run_plan(plan, **kw)


def test_library_loads_and_kernels_run():
    import torch
    from paper_2509_14098_b200 import kernels

    b = torch.zeros((1, 4), dtype=torch.complex128, device="cuda")
    b[0, 0] = 1
    h = np.array([[1, 1], [1, -1]], dtype=complex) / np.sqrt(2)
    kernels.apply_gate(b, h, [0])
    np.testing.assert_allclose(b.cpu().numpy()[0], [2 ** -0.5, 0, 2 ** -0.5, 0], atol=1e-15)


def test_grid_blocks_match_reference(grid_docs, grid_states):
    worst, n = 0.0, 0
    for doc in grid_docs:
        name = doc["name"]
        if name not in grid_states:
            continue
        res = _run(plan_from_doc(doc["plan"]))
        got = res.state.blocks.cpu().numpy()
        err = float(np.max(np.abs(got - grid_states[name])))
        assert err < TOL, (name, err)
        assert res.stats.task_counts == doc["stats"]["task_counts"], name
        assert res.stats.exchanges == doc["stats"]["exchanges"], name
        worst = max(worst, err)
        n += 1
    assert n >= 400
    print(f"grid parity: {n} cases, worst {worst:.2e}")


def test_grid_d12_matches_oracle(grid_docs):
    from oracle import oracle as orc

    n = 0
    for doc in grid_docs:
        if doc["plan"]["d"] != 12:
            continue
        plan = plan_from_doc(doc["plan"])
        ref, _ = orc.run_plan(plan, backend="numpy")
        got = _run(plan).state.blocks.cpu().numpy()
        assert np.max(np.abs(got - ref)) < TOL, doc["name"]
        n += 1
    assert n > 50


@pytest.mark.parametrize("key", ["18", "18_12"])
def test_cfg1_qft20_four_ranks(cfg1_docs, cfg1_fp, key):
    plan = plan_from_doc(cfg1_docs[key]["plan"])
    res = _run(plan)
    flat = res.state.blocks.reshape(-1).cpu().numpy()
    idx = cfg1_fp[key + "::idx"]
    assert np.max(np.abs(flat[idx] - cfg1_fp[key + "::amps"])) < TOL
    assert abs(flat.sum() - cfg1_fp[key + "::sum"][0]) < 1e-8
    assert res.state.layouts == cfg1_docs[key]["plan"]["layout_phases"]


def test_grid_jit_path_matches_reference(grid_docs, grid_states):
    """The NVRTC-specialised kernels on a slice of the grid (both code paths are product paths)."""
    n = 0
    for doc in grid_docs:
        name = doc["name"]
        if name not in grid_states or doc["plan"]["d"] < 8 or n >= 60:
            continue
        res = _run(plan_from_doc(doc["plan"]), jit=True)
        err = float(np.max(np.abs(res.state.blocks.cpu().numpy() - grid_states[name])))
        assert err < TOL, (name, err)
        n += 1
    assert n == 60


@pytest.mark.parametrize("key", ["18", "18_12"])
def test_cfg1_interpreter_path(cfg1_docs, cfg1_fp, key):
    plan = plan_from_doc(cfg1_docs[key]["plan"])
    flat = _run(plan, jit=False).state.blocks.reshape(-1).cpu().numpy()
    idx = cfg1_fp[key + "::idx"]
    assert np.max(np.abs(flat[idx] - cfg1_fp[key + "::amps"])) < TOL
