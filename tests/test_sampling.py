"""Device sampling (paper_2509_14098_b200/sampling.py) against numpy's
Generator.choice, the reference's sampler (svpart/executor.py:375-383).

CPU: (1) numpy's choice(p=...) is the CDF inversion sampling.py restates;
(2) the sharded algorithm -- basis-sorted shard probabilities, per-shard CDF
shares, a d-step binary search summed over shards -- replayed in numpy with
the kernels' index logic reproduces numpy's outcomes for random layouts and
shardings.  GPU: run_plan(shots=...) and sample() against numpy on the
gathered state.
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


def _shard_rank(m, d, fmask, fval):
    """Twin of shard_rank in csrc/sample.cu."""
    below = []
    c = 0
    for p in range(d):
        below.append(c)
        if not (fmask >> p) & 1:
            c += 1
    cnt = 0
    for p in range(d - 1, -1, -1):
        mb = (m >> p) & 1
        if (fmask >> p) & 1:
            fb = (fval >> p) & 1
            if mb > fb:
                return cnt + (1 << below[p])
            if mb < fb:
                return cnt
        elif mb:
            cnt += 1 << below[p]
    return cnt + 1


@pytest.mark.parametrize("d,g,world", [(5, 0, 1), (6, 2, 1), (6, 2, 2), (7, 3, 4), (7, 3, 8), (8, 2, 4)])
def test_sharded_sampling_replay(d, g, world):
    rng = np.random.default_rng(d * 100 + g * 10 + world)
    L = d - g
    rows = (1 << g) // world
    layout = list(rng.permutation(d))
    dense = rng.normal(size=1 << d) + 1j * rng.normal(size=1 << d)
    # storage order: dense[b(f)] = blocks.flat[f]
    f = np.arange(1 << d)
    b = np.zeros_like(f)
    for q in range(d):
        b |= ((f >> (d - 1 - layout[q])) & 1) << (d - 1 - q)
    flat = np.empty_like(dense)
    flat[f] = dense[b]
    shots, seed = 400, 1234
    u = np.random.default_rng(seed).random(shots)
    p_all = np.abs(dense) ** 2
    total = p_all.sum()
    shards = []
    for w in range(world):
        rank_base = w * rows
        D, perm, fmask, fval = sampling.shard_geometry(layout, d, g, rows, rank_base)
        shard = flat[(rank_base << L):(rank_base << L) + (1 << D)]
        sorted_p = np.empty(1 << D)
        t = np.arange(1 << D)
        j = np.zeros_like(t)
        for s in range(D):
            j |= ((t >> s) & 1) << perm[s]
        sorted_p[j] = np.abs(shard) ** 2
        # basis indices of the sorted shard must be increasing with the fixed bits applied
        bases = np.empty(1 << D, dtype=np.int64)
        bases[j] = b[(rank_base << L) + t]
        assert np.all(np.diff(bases) > 0)
        assert np.all((bases & fmask) == fval)
        shards.append((np.cumsum(sorted_p / total), fmask, fval))
    last = sum(c[-1] for c, _, _ in shards)
    lo = np.zeros(shots, dtype=np.int64)
    hi = np.full(shots, (1 << d) - 1, dtype=np.int64)
    for _ in range(d):
        mid = (lo + hi) // 2
        share = np.zeros(shots)
        for cdf, fmask, fval in shards:
            for s in range(shots):
                c = _shard_rank(int(mid[s]), d, fmask, fval)
                share[s] += cdf[c - 1] if c else 0.0
        take = share / last > u
        hi = np.where(take, mid, hi)
        lo = np.where(take, lo, mid + 1)
    want = np.random.default_rng(seed).choice(1 << d, size=shots, p=p_all / total)
    np.testing.assert_array_equal(lo, want)


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
