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


@pytest.mark.parametrize("world,kmax", [(1, 12), (1, 6), (1, 7), (2, 6), (4, 7)])
def test_sparse_start_programs_match_reference(grid_docs, grid_states, world, kmax):
    """Runs from |0...0> computing only the support (program.sparse_start):
    unwritten memory starts as NaN, so a read outside the support shows.
    Small tiles (kmax < D) give several sparse sweeps with dead tiles."""
    from paper_2509_14098_b200 import program as prog

    n = multi = 0
    for doc in _cases(grid_docs, grid_states, min_ranks=world):
        plan = plan_from_doc(doc["plan"])
        blocks, norms = program_emu.emulate_plan(plan, world=world, sparse=True, kmax=kmax)
        geo = prog.DeviceGeometry(d=plan.d, g=plan.g, h=plan.g - (world.bit_length() - 1), rank_base=0,
                                  pad_to=prog.RB)
        multi += len(prog.sparse_start(prog.plan_device(plan, geo, kmax=kmax), geo.D, True)) > 1
        err = float(np.max(np.abs(blocks - grid_states[doc["name"]])))
        assert err < TOL, (doc["name"], world, err)
        if world == 1:
            assert np.all(np.abs(norms - 1) < 1e-8), doc["name"]
        n += 1
    assert n > 50
    assert multi > (20 if kmax < 12 else -1)


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


def test_two_involutions_compose_to_the_permutation():
    """executor._two_involutions: any bit permutation as two passes of disjoint
    transpositions (the in-place initial-state layout change)."""
    import random

    from paper_2509_14098_b200.executor import _two_involutions

    rng = random.Random(5)

    def apply(pairs, r):
        for x, y in pairs:
            if r == x:
                return y
            if r == y:
                return x
        return r

    for n in range(1, 34):
        for _ in range(20):
            perm = list(range(n))
            rng.shuffle(perm)
            a, b = _two_involutions(perm)
            for pairs in (a, b):
                used = [x for p in pairs for x in p]
                assert len(used) == len(set(used))
            assert all(apply(b, apply(a, r)) == perm[r] for r in range(n))


def test_stable_thread_orders():
    """program._thread_orders(stable=True): a tile bit that stays a thread bit
    keeps its position; warp positions (>= 5) hold the bits needed last."""
    from paper_2509_14098_b200 import program as prog

    K = 12
    stages = [[{0, 1, 2, 3}, []], [{0, 1, 4, 5}, []], [{2, 3, 6, 7}, []], [{8, 9, 10, 11}, []]]
    orders = prog._thread_orders(stages, K, stable=True)
    for (rbits, _), order in zip(stages, orders):
        assert sorted(order) == [k for k in range(K) if k not in rbits]
    for prev, cur in zip(orders, orders[1:]):
        for p, k in enumerate(prev):
            if k in cur:
                assert cur[p] == k
    # stage 0: bits needed by later stages sit on lanes, never-needed-again ones on warp positions
    assert set(orders[0][5:]) <= {8, 9, 10, 11}
    assert prog.unpack_order(prog.pack_order(orders[2]), K - 4) == orders[2]
    assert prog._thread_orders(stages, K, stable=False)[1] == [2, 3, 6, 7, 8, 9, 10, 11]



@pytest.mark.parametrize("world,kmax,fold", [(2, 12, True), (4, 12, True), (2, 6, True), (4, 7, True),
                                             (8, 12, True), (2, 6, False), (4, 7, False)])
def test_localized_first_remap_matches_reference(grid_docs, grid_states, world, kmax, fold):
    """Runs from |0...0> whose first remap follows only sparse sweeps: every
    device computes the prefix as the unit-holding device and the remap is
    a local region move (program.localize_applies)."""
    from paper_2509_14098_b200 import program as prog

    n = used = 0
    for doc in _cases(grid_docs, grid_states, min_ranks=world):
        plan = plan_from_doc(doc["plan"])
        blocks, norms = program_emu.emulate_plan(plan, world=world, sparse=True, kmax=kmax, localize=True, fold=fold)
        err = float(np.max(np.abs(blocks - grid_states[doc["name"]])))
        assert err < TOL, (doc["name"], world, err)
        assert np.all(np.abs(norms - 1) < 1e-8), doc["name"]
        rows = (1 << plan.g) // world
        geo = prog.DeviceGeometry(d=plan.d, g=plan.g, h=rows.bit_length() - 1, rank_base=0, pad_to=prog.RB)
        used += prog.localize_applies(prog.plan_device(plan, geo, kmax=kmax), geo.D, world, geo.h)
        n += 1
    assert n > 20 and used > 5, (n, used)


@pytest.mark.parametrize("world,kmax", [(1, 12), (1, 6), (2, 12), (4, 12), (2, 6), (4, 7)])
def test_broadcast_merge_matches_reference(grid_docs, grid_states, world, kmax):
    """Runs from |0...0> with the broadcast merge (executor._broadcast_merges):
    a sweep that only expands dead bits is skipped and the sweep before it
    stores every value at all combinations of those bits (also across a
    folded localized remap), against the reference's blocks."""
    n = merged = 0
    for doc in _cases(grid_docs, grid_states, min_ranks=world):
        plan = plan_from_doc(doc["plan"])
        blocks, _ = program_emu.emulate_plan(plan, world=world, sparse=True, kmax=kmax, localize=world > 1,
                                             merge=True)
        err = float(np.max(np.abs(blocks - grid_states[doc["name"]])))
        assert err < TOL, (doc["name"], world, err)
        merged += program_emu.LAST_MERGES > 0
        n += 1
    assert n > 20, n
    if kmax < 12:  # the grid plans (d <= 12) fit one 12-bit tile otherwise
        assert merged > 0, (world, kmax)
    print(f"world {world} kmax {kmax}: {n} plans, {merged} with a merge")
