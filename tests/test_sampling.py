"""Device sampling (paper_2509_14098_b200/sampling.py) against numpy's
Generator.choice, the reference's sampler (svpart/executor.py:375-383).

CPU: (1) numpy's choice(p=...) is the CDF inversion sampling.py restates;
(2) the redistribution of sharded probabilities into contiguous basis
ranges, replayed in numpy, is exact for random layouts and shardings (the
floating-point steps are restated in tests/test_sampling_exact.py).  GPU:
run_plan(shots=...) and sample() against numpy on the gathered state, and
outcomes for adversarial uniforms on and next to every CDF boundary.
"""

import numpy as np
import pytest
import torch

from paper_2509_14098_b200 import sampling


def test_numpy_choice_is_cdf_inversion():
    for trial in range(10):
        rng0 = np.random.default_rng(trial)
        n = int(rng0.integers(2, 3000))
        a = rng0.normal(size=n) + 1j * rng0.normal(size=n)
        p = np.abs(a) ** 2
        p = p / p.sum()
        seed = int(rng0.integers(0, 1 << 30))
        want = np.random.default_rng(seed).choice(n, size=500, p=p)
        cdf = p.cumsum()
        cdf /= cdf[-1]
        got = cdf.searchsorted(np.random.default_rng(seed).random(500), side="right")
        np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("d,g,world", [(5, 0, 1), (6, 2, 1), (6, 2, 2), (7, 3, 4), (7, 3, 8), (8, 2, 4), (9, 3, 2)])
def test_basis_range_redistribution_replay(d, g, world):
    """sampling._to_basis_ranges replayed in numpy: every process's
    basis-sorted shard probabilities, sent with the planned splits and
    deposited with the planned bits, give each process exactly its
    contiguous range of the basis-order probability vector."""
    rng = np.random.default_rng(d * 100 + g * 10 + world)
    L = d - g
    rows = (1 << g) // world
    layout = list(rng.permutation(d))
    dense = rng.normal(size=1 << d) + 1j * rng.normal(size=1 << d)
    f = np.arange(1 << d)
    b = np.zeros_like(f)
    for q in range(d):
        b |= ((f >> (d - 1 - layout[q])) & 1) << (d - 1 - q)
    flat = np.empty_like(dense)
    flat[f] = dense[b]
    p_all = np.abs(dense) ** 2
    sorted_shards = []
    for w in range(world):
        rank_base = w * rows
        D, perm, fmask, fval = sampling.shard_geometry(layout, d, g, rows, rank_base)
        shard = flat[(rank_base << L):(rank_base << L) + (1 << D)]
        t = np.arange(1 << D)
        j = np.zeros_like(t)
        for s in range(D):
            j |= ((t >> s) & 1) << perm[s]
        sp = np.empty(1 << D)
        sp[j] = np.abs(shard) ** 2
        sorted_shards.append(sp)
    plans = [sampling.range_plan(layout, d, g, rows, world, me) for me in range(world)]
    # all_to_all_single: source p's send block for r arrives at r in source order
    sent = []
    for p in range(world):
        ins = plans[p][0]
        offs = np.cumsum([0] + ins)
        sent.append([sorted_shards[p][offs[r]:offs[r + 1]] for r in range(world)])
    n = 1 << (d - (world.bit_length() - 1))
    for me in range(world):
        recv = np.concatenate([sent[p][me] for p in range(world)])
        assert [len(sent[p][me]) for p in range(world)] == plans[me][1]
        q = np.full(n, np.nan)
        off = 0
        for low, or_val in plans[me][2]:
            cnt = 1 << len(low)
            t = np.arange(cnt)
            dst = np.full(cnt, or_val, dtype=np.int64)
            for i, bit in enumerate(low):
                dst |= ((t >> i) & 1) << bit
            q[dst] = recv[off:off + cnt]
            off += cnt
        np.testing.assert_array_equal(q, p_all[me * n:(me + 1) * n])


@pytest.mark.gpu
def test_device_sampling_matches_numpy():
    import gzip
    import json
    from pathlib import Path

    from paper_2509_14098_b200 import gather, plan as planmod, run_plan, sample

    docs = json.load(gzip.open(Path(__file__).parent / "golden" / "grid.json.gz", "rt"))
    checked = 0
    for doc in docs[::7]:
        plan = planmod.from_json(json.dumps(doc["plan"]))
        if plan.d < 3:
            continue
        seed = 1000 + checked
        res = run_plan(plan, shots=2000, seed=seed)
        dense = gather(res.state)
        p = np.abs(dense) ** 2
        outcomes = np.random.default_rng(seed).choice(len(dense), size=2000, p=p / p.sum())
        values, counts = np.unique(outcomes, return_counts=True)
        want = {format(int(v), f"0{plan.d}b"): int(c) for v, c in zip(values, counts)}
        assert res.histogram == want, doc["name"]
        assert sample(dense, 2000, seed) == want
        assert sample(torch.from_numpy(dense).cuda(), 2000, seed) == want
        checked += 1
    assert checked >= 20


@pytest.mark.gpu
def test_device_sampling_reference_known_answer():
    """sample(|10>) -> {"10": 50} (reference test_executor.py:140-143)."""
    from paper_2509_14098_b200 import sample

    assert sample(np.array([0, 0, 1, 0], dtype=np.complex128), 50, 0) == {"10": 50}


@pytest.mark.gpu
@pytest.mark.parametrize("d", [12, 20, 24])
def test_outcomes_identical_at_cdf_boundaries(d):
    """Uniforms exactly on, and one ulp either side of, CDF values: the
    device outcome equals numpy's searchsorted(cdf, u, "right") for every one
    (a parallel scan of the CDF would round some of these the other way)."""
    from paper_2509_14098_b200 import scatter
    from paper_2509_14098_b200.plan import ExecutionPlan

    rng = np.random.default_rng(d)
    a = rng.normal(size=1 << d) * np.exp(rng.uniform(-8, 0, size=1 << d)) + 1j * rng.normal(size=1 << d)
    a[rng.integers(0, 1 << d, 64)] = 0.0
    a /= np.linalg.norm(a)
    p = np.abs(a) ** 2
    p = p / p.sum()
    cdf = p.cumsum()
    cdf /= cdf[-1]
    idx = rng.integers(0, 1 << d, 3000)
    u = np.concatenate([cdf[idx], np.nextafter(cdf[idx], 0.0), np.nextafter(cdf[idx], 2.0),
                        [0.0, np.nextafter(1.0, 0.0), 0.5], rng.random(2000)])
    u = u[(u >= 0.0) & (u < 1.0)]
    want = cdf.searchsorted(u, side="right")
    plan = ExecutionPlan(d, 0, [list(range(d))], [])
    st = scatter(a, plan)
    got = sampling.outcomes(st, u).cpu().numpy()
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (bad[:10], got[bad[:10]], want[bad[:10]])
    # and whole histograms through the public API
    from paper_2509_14098_b200 import sample

    for seed in (1, 2):
        outc = np.random.default_rng(seed).choice(1 << d, size=20000, p=p)
        vals, cnts = np.unique(outc, return_counts=True)
        assert sample(a, 20000, seed) == {format(int(v), f"0{d}b"): int(c) for v, c in zip(vals, cnts)}
