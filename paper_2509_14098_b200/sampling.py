"""Measurement sampling on the device (svpart/executor.py:375-383).

The reference gathers the state to the host and calls
``default_rng(seed).choice(2^d, shots, p=|psi|^2 / sum)``.  numpy evaluates
that as (checked in tests/test_sampling.py)::

    cdf = cumsum(p); cdf /= cdf[-1]; u = rng.random(shots)
    outcome = searchsorted(cdf, u, side="right")        # over the basis order

Here the uniforms are drawn by the same numpy Generator on the host (shots x
8 bytes), and everything of size 2^d stays on the GPUs, sharded as the state
is:

1. each process writes |a|^2 of its shard in basis-sorted shard order
   (``svb_probs_sorted``) and normalises by the all-reduced sum;
2. an inclusive scan of that array gives the shard's share of the CDF at any
   of its own elements;
3. a binary search over [0, 2^d) runs for all shots at once: at each of the
   d steps every process evaluates its share of the CDF at the shots'
   candidate indices (``svb_sample_prefix``), the shares are all-reduced and
   compared with u.

Outcomes equal the reference's except when a uniform falls within a few
ulps of a CDF boundary, where the different summation order (tree sums and a
parallel scan instead of numpy's pairwise sum and sequential cumsum) can
round the other way.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native


def shard_geometry(layout, d: int, g: int, rows: int, rank_base: int):
    """(D, perm, fixed_mask, fixed_val) of a process's shard.

    The shard holds global storage indices (rank_base << L) + t, t < 2^D,
    D = L + log2(rows).  Storage bit s (LSB-indexed) is basis bit
    bp[s] = d-1-q for the qubit q with layout[q] = d-1-s.  perm[s] is the rank
    of bp[s] among the shard's free basis bits (its bit in basis-sorted shard
    order); the other basis bits are fixed by the shard's top rank bits.
    """
    L = d - g
    h = rows.bit_length() - 1
    D = L + h
    bp = [0] * d
    for q in range(d):
        bp[d - 1 - layout[q]] = d - 1 - q
    free = sorted(bp[s] for s in range(D))
    pos = {b: i for i, b in enumerate(free)}
    perm = [pos[bp[s]] for s in range(D)]
    fixed_mask = fixed_val = 0
    for s in range(D, d):
        fixed_mask |= 1 << bp[s]
        if ((rank_base << L) >> s) & 1:
            fixed_val |= 1 << bp[s]
    return D, perm, fixed_mask, fixed_val


def sample_state(state, shots: int, seed: int | None) -> dict:
    """Seeded histogram {bitstring: count} of a (possibly sharded) DistState,
    qubit 0 first, computed on the GPU(s).  Collective when sharded."""
    lib = _native.load()
    d, g = state.d, state.g
    blocks = state.blocks
    device = blocks.device
    rows = blocks.shape[0]
    world = state.world
    D, perm, fmask, fval = shard_geometry(state.layouts[state.phase], d, g, rows, state.rank_base)

    def allsum(t):
        if world > 1:
            import torch.distributed as dist

            dist.all_reduce(t, group=state.group)
        return t

    stream = torch.cuda.current_stream(device).cuda_stream
    need = 8 << D  # |a|^2 of the shard, float64
    free, _ = torch.cuda.mem_get_info(device)
    if need + (1 << 30) > free + torch.cuda.memory_reserved(device) - torch.cuda.memory_allocated(device):
        from .errors import TooLarge

        raise TooLarge(f"sampling needs {need >> 30} GiB of probabilities beside the state on {device} "
                       f"({free >> 30} GiB free): run on more GPUs or sample a gathered sub-state")
    probs = torch.empty(1 << D, dtype=torch.float64, device=device)
    arr, p32 = _native.i32_array(perm)
    _native.check(lib.svb_probs_sorted(blocks.contiguous().data_ptr(), D, p32, probs.data_ptr(), stream),
                  "svb_probs_sorted")
    total = allsum(probs.sum().reshape(1))
    probs /= total  # numpy: probs = probs / probs.sum()
    cdf = probs.cumsum_(0)  # this shard's share of the CDF, in basis order
    last = allsum(cdf[-1:].clone())  # numpy: cdf /= cdf[-1]
    u = torch.from_numpy(np.random.default_rng(seed).random(shots)).to(device)
    lo = torch.zeros(shots, dtype=torch.int64, device=device)
    hi = torch.full((shots,), (1 << d) - 1, dtype=torch.int64, device=device)
    share = torch.empty(shots, dtype=torch.float64, device=device)
    for _ in range(d):  # smallest i with cdf[i] / cdf[-1] > u (searchsorted, side="right")
        mid = (lo + hi) // 2
        _native.check(lib.svb_sample_prefix(cdf.data_ptr(), d, fmask, fval, mid.data_ptr(), shots,
                                            share.data_ptr(), stream), "svb_sample_prefix")
        take = allsum(share) / last > u
        hi = torch.where(take, mid, hi)
        lo = torch.where(take, lo, mid + 1)
    del cdf, probs
    values, counts = torch.unique(lo, return_counts=True)
    return {format(int(v), f"0{d}b"): int(c) for v, c in zip(values.tolist(), counts.tolist())}
