"""CPU validation of the host compiler + layout planner through the kernel emulator."""

import numpy as np
import pytest

from conftest import plan_from_doc
import program_emu

TOL = 1e-10


def _cases(grid_docs, grid_states, limit=None, min_ranks=1):
    out = []
    for doc in grid_docs:
        if doc["name"] in grid_states and (1 << doc["plan"]["g"]) >= min_ranks:
            out.append(doc)
    return out[:limit] if limit else out


@pytest.mark.parametrize("rb,stable", [(4, False), (3, False), (4, True)])
def test_single_device_programs_match_reference(grid_docs, grid_states, rb, stable):
    """stable=True: planner-chosen thread-bit orders (the generated kernels' layout)."""
    worst = 0.0
    for doc in _cases(grid_docs, grid_states):
        plan = plan_from_doc(doc["plan"])
        blocks, norms = program_emu.emulate_plan(plan, rb=rb, stable=stable)
        err = float(np.max(np.abs(blocks - grid_states[doc["name"]])))
        assert err < TOL, (doc["name"], err)
        assert np.all(np.abs(norms - 1) < 1e-8), doc["name"]
        worst = max(worst, err)
    print("worst", worst)


@pytest.mark.parametrize("world", [2, 4])
def test_multi_device_programs_match_reference(grid_docs, grid_states, world):
    n = 0
    for doc in _cases(grid_docs, grid_states, min_ranks=world):
        plan = plan_from_doc(doc["plan"])
        blocks, _ = program_emu.emulate_plan(plan, world=world)
        err = float(np.max(np.abs(blocks - grid_states[doc["name"]])))
        assert err < TOL, (doc["name"], world, err)
        n += 1
    assert n > 50
