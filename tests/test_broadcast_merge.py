"""Broadcast merge (executor._broadcast_merges): a sparse sweep that only
expands never-touched qubits (H on dead bits, one constant scale) is folded
into the store of the sweep before it."""

from pathlib import Path

import numpy as np
import pytest

PLANS = Path(__file__).resolve().parent.parent / "plans"


def load(name):
    from paper_2509_14098_b200 import plan as planmod

    return planmod.load(str(PLANS / f"{name}.json.gz"))


def merges(name):
    from paper_2509_14098_b200 import executor as ex, program as prog

    plan = load(name)
    geo = prog.DeviceGeometry(d=plan.d, g=plan.g, h=plan.g, rank_base=0, pad_to=prog.RB)
    dp = prog.plan_device(plan, geo, rb=4, overlap_bits=0, free_start=True, stable_threads=False)
    sparse = prog.sparse_start(dp, geo.D, True)
    return dp, sparse, ex._broadcast_merges(dp, geo, sparse, {}, {}, {})


def test_qft30_last_sweep_is_a_broadcast_of_two_qubits():
    """QFT-30's last sweep only applies H to qubits 28 and 29, which no
    earlier gate touched: it merges into sweep 2 with F = {28, 29} and the
    scale of the two H gates; sweep 2 keeps its own leaf norm and adds the
    merged leaf's at the other slot."""
    dp, sparse, bc = merges("qft30_h30-12")
    assert set(bc) == {2}
    fmask, copies, off, slot = bc[2]
    assert fmask == (1 << 28) | (1 << 29)
    assert sorted(copies) == [0, 1 << 28, 1 << 29, 3 << 28]
    assert all(len(ch) == 1 and abs(ch[0] - 0.5) < 1e-15 for ch in copies.values())
    assert slot == int(dp.buf.descs[2]["norm_slot"]) and off == int(dp.buf.descs[3]["norm_slot"]) - slot
    # the merged sweep wrote only the support; the broadcast covers the rest
    supp, full_out = sparse[3]
    assert full_out and supp | fmask == (1 << 30) - 1


def test_no_merge_when_the_sweep_computes():
    """QV and a sweep that mixes live amplitudes never merge."""
    _, _, bc = merges("qv30_h30-12")
    assert bc == {}


def test_merge_source_stores_every_combination():
    from paper_2509_14098_b200 import jit

    dp, sparse, bc = merges("qft22_h22-12")
    (j, (fmask, copies, off, slot)), = bc.items()
    d = dp.buf.descs[j]
    ops = dp.buf.ops[d["op_begin"]: d["op_begin"] + d["op_count"]]
    src = jit.kernel_source("k", d, ops, dp.buf.coef, 0, sparse[j], 0, None, bc[j])
    nf = bin(fmask).count("1")
    stores = src.count("st_stream(")
    plain = jit.kernel_source("k", d, ops, dp.buf.coef, 0, sparse[j]).count("st_stream(")
    assert stores == plain * (1 << nf)


def test_multi_gpu_merges_cross_the_folded_localize():
    """On 2 and 4 GPUs the last prefix sweep keeps region alpha and the
    sweep after the folded localized remap only expands the swapped bits
    (on 4 GPUs a fused 4x4 on them, with the final relabel of the two bits):
    both merge, for every rank."""
    from paper_2509_14098_b200 import executor as ex, program as prog

    for name, world in (("qft31_h30-12", 2), ("qft32_h30-12", 4)):
        plan = load(name)
        rows = (1 << plan.g) // world
        for me in range(world):
            geo = prog.DeviceGeometry(d=plan.d, g=plan.g, h=rows.bit_length() - 1, rank_base=me * rows,
                                      pad_to=prog.RB)
            dp0 = prog.plan_device(plan, geo, rb=4, overlap_bits=0, free_start=True, stable_threads=False)
            rep = prog.localize_applies(dp0, geo.D, world, geo.h)
            assert rep
            dp = prog.plan_device(plan, geo, rb=4, overlap_bits=0, free_start=True, stable_threads=False,
                                  overlap_skip_first=True, replicate_prefix=True)
            sparse = prog.sparse_start(dp, geo.D, True)
            ldx = ex._fold_localize(dp, geo, sparse)
            stk = ex._prefix_store_masks(dp, geo, sparse)
            bc = ex._broadcast_merges(dp, geo, sparse, ldx, stk, {})
            assert len(bc) == 1, (name, me)
            (j, (fmask, copies, off, slot)), = bc.items()
            assert bin(fmask).count("1") == world.bit_length() - 1
            assert len(copies) == world


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["qft22_h22-12", "qft28_h28-12", "qft30_h30-12"])
def test_merged_equals_unmerged_and_closed_form(name):
    """Merged and unmerged runs give equal amplitudes and norms, and QFT|0>
    is the uniform state 2^-d/2 (every broadcast position written)."""
    import torch

    from paper_2509_14098_b200 import executor, run_plan

    plan = load(name)
    a = run_plan(plan)
    sa = a.stats.sweeps
    blocks_a = a.state.blocks
    executor.BROADCAST_MERGE = False
    executor._compile_cache.clear()
    try:
        b = run_plan(plan)
        assert torch.equal(blocks_a, b.state.blocks), name
        assert b.stats.sweeps == sa + 1
    finally:
        executor.BROADCAST_MERGE = True
        executor._compile_cache.clear()
    u = 2.0 ** (-plan.d / 2)
    err = (blocks_a - u).abs().max().item()
    assert err < 1e-12, (name, err)
    assert np.isfinite(err)


@pytest.mark.gpu
def test_merged_plan_against_the_oracle():
    """QFT-22 from |0...0> (its last sweep merges) against the CPU
    restatement of the reference executor, every amplitude."""
    import os

    from oracle import oracle as orc
    from paper_2509_14098_b200 import run_plan

    plan = load("qft22_h22-12")
    res = run_plan(plan)
    dp, _, bc = merges("qft22_h22-12")
    assert res.stats.sweeps == len(dp.buf.descs) - len(bc)
    got = res.state.blocks.cpu().numpy()
    ref, _ = orc.run_plan(plan, backend="c", nthreads=os.cpu_count() or 1)
    assert np.max(np.abs(got - ref)) < 1e-12
