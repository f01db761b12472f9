"""8-GPU readiness without 8 GPUs: the device programs of all eight ranks of
the 8-GPU benchmark configs (BASELINE cfg3 QV-34 [31,12], cfg4 QAOA-35
[32,12], cfg5 SUP-36 [33,12]) are compiled here and checked for the
properties the run relies on (plan.py:59-75, executor.py:250-268)."""

import numpy as np
import pytest

from conftest import ROOT

from paper_2509_14098_b200 import comm, plan as planmod, program as prog

HBM_BYTES = 179 << 30  # B200: 183,359 MiB reported; keep 1 GiB+ for the runtime
WORLD = 8


def _programs(name):
    plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
    rows = (1 << plan.g) // WORLD
    out = []
    for w in range(WORLD):
        geo = prog.DeviceGeometry(d=plan.d, g=plan.g, h=rows.bit_length() - 1, rank_base=w * rows, pad_to=prog.RB)
        out.append((geo, prog.plan_device(plan, geo, rb=4, overlap_bits=3)))
    return plan, out


@pytest.mark.parametrize("name", ["sup36_h33-12", "qaoa35_h32-12", "qv34_h31-12"])
def test_eight_rank_programs(name):
    plan, progs = _programs(name)
    assert (1 << plan.g) == WORLD  # one rank per GPU
    ref = [(s.kind, s.task_id, s.swaps, s.cbits, s.first, s.count) for s in progs[0][1].steps]
    for geo, dp in progs[1:]:  # every process derives the same schedule and layouts
        assert [(s.kind, s.task_id, s.swaps, s.cbits, s.first, s.count) for s in dp.steps] == ref
        assert dp.init_perm == progs[0][1].init_perm
        assert dp.norm_alias == progs[0][1].norm_alias
    geo0 = progs[0][0]
    # memory: the state (one rank of 2^L amplitudes) plus the flag words of
    # the peer remap; the remap is in place, so nothing else scales with L
    state = 16 << geo0.L
    assert state + comm.FLAG_BYTES <= HBM_BYTES, (name, state >> 30)
    # the sparse |0...0> start: rank 0 holds the unit vector, the others zeros
    for w, (geo, dp) in enumerate(progs):
        sp = prog.sparse_start(dp, geo.D, w == 0)
        if w:
            assert all(s is None for s, _ in sp.values())
    # exchanges: 2^m - 1 partners, and each round of the partner order is a
    # perfect matching of the 8 processes
    ex = [s for s in progs[0][1].steps if s.kind == "exchange" and s.swaps]
    assert len(ex) == sum(1 for t in plan.tasks if t.kind == "Exchange")
    for st in ex:
        m = len(st.swaps)
        ebits = [ib for ib, _ in st.swaps]
        rounds = {}
        for me in range(WORLD):
            pp = comm.peer_plan(me, ebits, m)
            assert len(pp) == (1 << m) - 1
            assert len({p.peer for p in pp}) == (1 << m) - 1 and me not in {p.peer for p in pp}
            alpha = 0
            for e in ebits:
                alpha = (alpha << 1) | ((me >> e) & 1)
            for r, p in enumerate(sorted(pp, key=lambda p: p.sel ^ alpha)):
                rounds.setdefault(r, {})[me] = p.peer
        for r, mate in rounds.items():
            assert all(mate[mate[me]] == me for me in mate), (name, r)
    if name == "sup36_h33-12":  # cfg5: one 3-bit remap per exchange, 7 partners each
        assert all(len(s.swaps) == 3 for s in ex)


def test_eight_rank_emulation(grid_docs, grid_states):
    """World-8 device programs on the reference grid (8-rank plans), executed
    by the kernel emulator with the remaps as physical bit swaps."""
    import program_emu
    from conftest import plan_from_doc

    n = 0
    for doc in grid_docs:
        if doc["name"] not in grid_states or (1 << doc["plan"]["g"]) < WORLD:
            continue
        plan = plan_from_doc(doc["plan"])
        blocks, _ = program_emu.emulate_plan(plan, world=WORLD)
        assert np.max(np.abs(blocks - grid_states[doc["name"]])) < 1e-10, doc["name"]
        n += 1
    assert n > 30
