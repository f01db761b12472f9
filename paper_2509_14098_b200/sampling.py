"""Measurement sampling on the device (svpart/executor.py:375-383), identical
to numpy by construction.

The reference gathers the state to the host and calls
``default_rng(seed).choice(2^d, shots, p=|psi|^2 / sum)``.  numpy evaluates
that as (checked in tests/test_sampling.py)::

    probs = np.abs(psi) ** 2; probs = probs / probs.sum()     # pairwise sum
    cdf = cumsum(probs); cdf /= cdf[-1]; u = rng.random(shots) # sequential cumsum
    outcome = searchsorted(cdf, u, side="right")              # basis order

Every floating-point step is reproduced bit for bit on the GPU(s)
(csrc/cdf.cu): numpy's complex absolute value, its pairwise summation tree,
the SEQUENTIAL cumsum (evaluated exactly through integer ulp increments per
binade, see cdf.cu), the normalisation and the right-sided search.  The
uniforms come from the same numpy Generator on the host (8 B per shot).

Sharded states: each process first writes |a|^2 of its shard in basis-sorted
shard order, then an all-to-all leaves process j with the contiguous basis
range [j 2^D, (j+1) 2^D) (a 2^D-element half of the state's bytes moves; the
state itself stays put).  The pairwise sum of the whole vector is the
pairwise tree over the processes' range sums (ranges are aligned halves of
the recursion), the exact cumsum is walked range after range (each process
starts from its predecessor's exact end value), and the shots are resolved
by the process owning their chunk.
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


def _free_bits(d: int, fixed_mask: int) -> list:
    return [b for b in range(d) if not (fixed_mask >> b) & 1]


def pairwise_combine(parts: list) -> float:
    """numpy's pairwise recursion over equal aligned ranges: a binary tree
    of left + right (python floats are IEEE doubles)."""
    vals = [float(x) for x in parts]
    while len(vals) > 1:
        vals = [vals[i] + vals[i + 1] for i in range(0, len(vals), 2)]
    return vals[0]


def sample_state(state, shots: int, seed: int | None) -> dict:
    """Seeded histogram {bitstring: count} of a (possibly sharded) DistState,
    qubit 0 first, computed on the GPU(s), equal to the reference's
    ``sample(gather(state), shots, seed)``.  Collective when sharded."""
    u = np.random.default_rng(seed).random(shots)
    out = outcomes(state, u)
    values, counts = torch.unique(out, return_counts=True)
    return {format(int(v), f"0{state.d}b"): int(c) for v, c in zip(values.tolist(), counts.tolist())}


def outcomes(state, u) -> torch.Tensor:
    """Basis indices numpy's choice(2^d, p=|psi|^2/sum) returns for the
    uniforms u (searchsorted(cdf, u, side="right")), as a device tensor."""
    import ctypes

    lib = _native.load()
    d, g = state.d, state.g
    blocks = state.blocks
    device = blocks.device
    rows = blocks.shape[0]
    world = state.world
    layout = state.layouts[state.phase]
    D, perm, fmask, fval = shard_geometry(layout, d, g, rows, state.rank_base)
    me = state.rank_base // rows
    stream = torch.cuda.current_stream(device).cuda_stream
    need = (8 << D) * (2 if world > 1 else 1)  # |a|^2 (+ the received range)
    free, _ = torch.cuda.mem_get_info(device)
    if need + (1 << 30) > free + torch.cuda.memory_reserved(device) - torch.cuda.memory_allocated(device):
        from .errors import TooLarge

        raise TooLarge(f"sampling needs {need >> 30} GiB of probabilities beside the state on {device} "
                       f"({free >> 30} GiB free): run on more GPUs or sample a gathered sub-state")

    def check(rc, what):
        _native.check(rc, what)

    p_local = torch.empty(1 << D, dtype=torch.float64, device=device)
    arr, p32 = _native.i32_array(perm)
    check(lib.svb_probs_numpy(blocks.contiguous().data_ptr(), D, p32, p_local.data_ptr(), stream), "svb_probs_numpy")
    if world > 1:
        q = _to_basis_ranges(state, p_local, D, d, g, rows, me, world, layout)
        del p_local
    else:
        q = p_local
    n = q.numel()
    # probs.sum(): numpy's pairwise sum of the whole vector
    ssum = torch.empty(1, dtype=torch.float64, device=device)
    scratch = torch.empty(int(lib.svb_pairwise_scratch_bytes(D)) // 8 + 1, dtype=torch.float64, device=device)
    check(lib.svb_pairwise_sum(q.data_ptr(), D, ssum.data_ptr(), scratch.data_ptr(), stream), "svb_pairwise_sum")
    if world > 1:
        parts = _all_gather_f64(ssum, world, state.group)
        total = pairwise_combine(parts)
        ssum.fill_(total)
    total = float(ssum.item())
    if not np.isfinite(total):
        raise ValueError("probabilities contain NaN")
    check(lib.svb_div_scalar(q.data_ptr(), n, ssum.data_ptr(), stream), "svb_div_scalar")
    # exact sequential cumsum: chunk classification from an approximate prefix,
    # then the walk from the exact start (the previous range's exact end)
    B = int(lib.svb_cdf_chunk_elems())
    nch = (n + B - 1) // B
    tot = torch.empty(nch, dtype=torch.float64, device=device)
    check(lib.svb_cdf_chunk_totals(q.data_ptr(), n, tot.data_ptr(), stream), "svb_cdf_chunk_totals")
    offset = 0.0
    if world > 1:
        mine = tot.sum().reshape(1)
        offset = float(sum(_all_gather_f64(mine, world, state.group)[:me]))
    cstart = torch.cumsum(tot, 0) - tot + offset
    fn = torch.empty(int(lib.svb_cdf_scratch_bytes(n)) // 8 + 1, dtype=torch.float64, device=device)
    cend = torch.empty(nch, dtype=torch.float64, device=device)
    nslow = torch.zeros(1, dtype=torch.int64, device=device)
    c_in = torch.zeros(1, dtype=torch.float64, device=device)
    for j in range(world):
        if j == me:
            check(lib.svb_cdf_walk(q.data_ptr(), n, cstart.data_ptr(), tot.data_ptr(), fn.data_ptr(),
                                   c_in.data_ptr(), cend.data_ptr(), nslow.data_ptr(), stream), "svb_cdf_walk")
        if world > 1:
            import torch.distributed as dist

            ex = cend[-1:].clone() if j == me else torch.empty(1, dtype=torch.float64, device=device)
            _broadcast(ex, j, state.group)
            if me == j + 1:
                c_in.copy_(ex)
    cend_all = torch.cat(_all_gather_tensor(cend, world, state.group)) if world > 1 else cend
    c_last = float(cend_all[-1].item())
    u = torch.as_tensor(np.ascontiguousarray(u, dtype=np.float64)).to(device)
    shots = u.numel()
    out = torch.empty(shots, dtype=torch.int64, device=device)
    check(lib.svb_cdf_search(q.data_ptr(), n, cend_all.data_ptr(), cend_all.numel(), me * nch, (me + 1) * nch,
                             ctypes.c_double(c_last), u.data_ptr(), shots, me * n, out.data_ptr(), stream),
          "svb_cdf_search")
    if world > 1:
        out = _all_reduce_max_i64(out, state.group)
    return out


def _gloo(group) -> bool:
    import torch.distributed as dist

    return dist.get_backend(group) == "gloo"


def _all_gather_tensor(t: torch.Tensor, world: int, group) -> list:
    import torch.distributed as dist

    if _gloo(group):  # gloo: through host memory
        h = t.cpu()
        parts = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(parts, h, group=group)
        return [p.to(t.device) for p in parts]
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return parts


def _all_gather_f64(t: torch.Tensor, world: int, group) -> list:
    return [float(x.item()) for x in _all_gather_tensor(t, world, group)]


def _broadcast(t: torch.Tensor, src: int, group) -> None:
    import torch.distributed as dist

    if _gloo(group):
        h = t.cpu()
        dist.broadcast(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src, group=group)


def _all_reduce_max_i64(t: torch.Tensor, group) -> torch.Tensor:
    import torch.distributed as dist

    if _gloo(group):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        return h.to(t.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def range_plan(layout, d: int, g: int, rows: int, world: int, me: int):
    """The all-to-all of _to_basis_ranges for process `me`: its send split
    per destination (its basis-sorted shard is grouped by destination), its
    receive split per source, and per source the basis bits below the
    range bits its elements enumerate plus the fixed low value they carry."""
    hb = world.bit_length() - 1
    top = list(range(d - hb, d))
    low_mask = (1 << (d - hb)) - 1

    def geo(p):
        D, _, fm, fv = shard_geometry(layout, d, g, rows, p * rows)
        free = _free_bits(d, fm)
        return D, fm, fv, free, [b for b in free if b >= d - hb]

    def sends_to(fm_, fv_, r):
        rb = r << (d - hb)
        return all(((rb >> b) & 1) == ((fv_ >> b) & 1) for b in top if (fm_ >> b) & 1)

    D, fm, fv, free, ftop = geo(me)
    in_splits = [(1 << (D - len(ftop))) if sends_to(fm, fv, r) else 0 for r in range(world)]
    out_splits, sources = [], []
    for p in range(world):
        pD, pfm, pfv, pfree, pftop = geo(p)
        ok = sends_to(pfm, pfv, me)
        out_splits.append((1 << (pD - len(pftop))) if ok else 0)
        if ok:
            sources.append(([b for b in pfree if b < d - hb], pfv & low_mask))
    return in_splits, out_splits, sources


def _to_basis_ranges(state, p_local, D, d, g, rows, me, world, layout) -> torch.Tensor:
    """All-to-all from basis-sorted shards to contiguous basis ranges:
    process j receives every |a|^2 whose top log2(world) basis bits read j,
    placed at its basis index below those bits (svb_deposit_scatter)."""
    import torch.distributed as dist

    lib = _native.load()
    in_splits, out_splits, sources = range_plan(layout, d, g, rows, world, me)
    assert sum(in_splits) == (1 << D) and sum(out_splits) == (1 << D)
    if _gloo(state.group):
        src_h = p_local.cpu()
        recv_h = torch.empty(1 << D, dtype=torch.float64)
        dist.all_to_all_single(recv_h, src_h, out_splits, in_splits, group=state.group)
        recv = recv_h.to(p_local.device)
    else:
        recv = torch.empty(1 << D, dtype=torch.float64, device=p_local.device)
        dist.all_to_all_single(recv, p_local, out_splits, in_splits, group=state.group)
    q = torch.empty(1 << D, dtype=torch.float64, device=p_local.device)
    stream = torch.cuda.current_stream(p_local.device).cuda_stream
    off = 0
    for low, or_val in sources:
        cnt = 1 << len(low)
        arr, bits32 = _native.i32_array(low)
        _native.check(lib.svb_deposit_scatter(recv[off:].data_ptr(), cnt, len(low), bits32, or_val,
                                              q.data_ptr(), stream), "svb_deposit_scatter")
        off += cnt
    return q
