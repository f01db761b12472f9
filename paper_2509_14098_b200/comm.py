"""Inter-GPU qubit remap: the Pack -> Exchange -> Unpack of executor.py:224-281
when the swapped rank bits select different GPUs.

With one process per GPU, a swap of device-id bit e_i with local bit l_i
(i < m) is a pairwise in-place exchange: process w, whose id reads alpha at
the e bits, trades its region {local l-bits = v} with peer w[e := v] for
every v != alpha, and the peer's data lands in that same region (derivation
in DESIGN.md "Remap").  Regions are not contiguous in general, so each
chunk is packed into a staging buffer by a CUDA kernel, moved with grouped
NCCL send/recv (all 2^m - 1 peers in one group), and unpacked; chunks are
double-buffered so packing chunk c+1 overlaps the transfer of chunk c.

The data movement functions are injectable so the protocol can be tested
with the gloo backend on CPU tensors (tests/test_comm_gloo.py).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

# NCCL send/recv on B200 NVLink is message-size bound (measured with
# tools/nvlink_bench.py: 298 GB/s at 64 MiB, 333 at 256 MiB, 636 at 1 GiB per
# direction), so chunks are as large as the staging budget allows.
STAGING_BYTES = int(os.environ.get("SVB200_STAGING_BYTES", str(8 << 30)))
MIN_CHUNK_BYTES = 256 << 20


@dataclass
class PeerPlan:
    peer: int  # process rank in the group
    sel: int  # region selector over the swapped local bits (bit m-1-i <-> lbits[i])


def peer_plan(me: int, ebits: list, m: int) -> list:
    """Peers and region selectors for one exchange, ascending by selector."""
    alpha = 0
    for e in ebits:
        alpha = (alpha << 1) | ((me >> e) & 1)
    out = []
    for v in range(1 << m):
        if v == alpha:
            continue
        peer = me
        for i, e in enumerate(ebits):
            bit = (v >> (m - 1 - i)) & 1
            peer = (peer | (1 << e)) if bit else (peer & ~(1 << e))
        out.append(PeerPlan(peer, v))
    return out


class CudaMover:
    """Pack/unpack through libsvb200 on the current CUDA stream."""

    def __init__(self, state):
        from . import _native

        self.lib = _native.load()
        self.state = state
        self._native = _native

    def pack(self, lbits, m, sel, off, count, out: torch.Tensor) -> None:
        arr, ptr = self._native.i32_array(lbits)
        st = torch.cuda.current_stream(out.device).cuda_stream
        self._native.check(
            self.lib.svb_pack_region(self.state.buf.data_ptr(), self.state.rows, self.state.L, ptr, m,
                                     sel, off, count, out.data_ptr(), st),
            "svb_pack_region",
        )

    def unpack(self, lbits, m, sel, off, count, inp: torch.Tensor) -> None:
        arr, ptr = self._native.i32_array(lbits)
        st = torch.cuda.current_stream(inp.device).cuda_stream
        self._native.check(
            self.lib.svb_unpack_region(self.state.buf.data_ptr(), self.state.rows, self.state.L, ptr,
                                       m, sel, off, count, inp.data_ptr(), st),
            "svb_unpack_region",
        )


def _as_real(t: torch.Tensor) -> torch.Tensor:
    return torch.view_as_real(t).reshape(-1) if t.is_complex() else t


def exchange(state, remote: list, geo, group, mover=None, chunk_elems: int | None = None,
             cbits: list | None = None, cval: int = 0) -> int:
    """Run one inter-process exchange; returns the number of kernel launches issued.

    `remote` lists (device-id bit, local device bit) pairs; `state` has
    .rows, .L and a flat complex128 `.buf` of rows * 2^L amplitudes.  With
    `cbits` only the part of every region whose chunk bits read `cval`
    (cbits[0] is its most significant bit) is exchanged, so a remap can be
    split into parts that overlap the sweeps around it.
    """
    import torch.distributed as dist

    me = dist.get_rank(group)
    m = len(remote)
    ebits = [e for e, _ in remote]
    cbits = list(cbits or [])
    k = len(cbits)
    lbits = [lb for _, lb in remote] + cbits
    peers = [PeerPlan(pp.peer, (pp.sel << k) | cval) for pp in peer_plan(me, ebits, m)]
    m = m + k  # selector width over lbits
    region = state.rows << (state.L - m)
    if chunk_elems is None:
        nbuf_bytes = max(MIN_CHUNK_BYTES, STAGING_BYTES // (2 * max(1, len(peers))))
        chunk_elems = max(1, min(region, nbuf_bytes // 16))
    mover = mover or CudaMover(state)
    dev = state.buf.device
    L = state.L
    # contiguous fast path: the swapped local bits are the top physical bits,
    # so every region is one contiguous block that NCCL can send in place
    contiguous = state.rows == 1 and sorted(lbits) == list(range(L - m, L))
    nbuf = 2
    send = [torch.empty((len(peers), chunk_elems), dtype=torch.complex128, device=dev)
            for _ in range(nbuf)] if not contiguous else None
    recv = [torch.empty((len(peers), chunk_elems), dtype=torch.complex128, device=dev) for _ in range(nbuf)]
    launches = 0
    nchunks = (region + chunk_elems - 1) // chunk_elems

    def region_base(sel):
        base = 0
        for i, lb in enumerate(lbits):
            if (sel >> (m - 1 - i)) & 1:
                base |= 1 << lb
        return base

    def issue(c):
        nonlocal launches
        off = c * chunk_elems
        cnt = min(chunk_elems, region - off)
        b = c % nbuf
        srcs = []
        for j, pp in enumerate(peers):
            if contiguous:
                a0 = region_base(pp.sel) + off
                srcs.append(state.buf[a0:a0 + cnt])
            else:
                mover.pack(lbits, m, pp.sel, off, cnt, send[b][j])
                launches += 1
                srcs.append(send[b][j, :cnt])
        ops = []
        for j, pp in enumerate(peers):
            ops.append(dist.P2POp(dist.isend, _as_real(srcs[j]), pp.peer, group))
            ops.append(dist.P2POp(dist.irecv, _as_real(recv[b][j, :cnt]), pp.peer, group))
        return dist.batch_isend_irecv(ops), off, cnt, b

    pending = issue(0) if nchunks else None
    for c in range(nchunks):
        nxt = issue(c + 1) if c + 1 < nchunks else None
        works, off, cnt, b = pending
        for w in works:
            w.wait()
        for j, pp in enumerate(peers):
            if contiguous:
                a0 = region_base(pp.sel) + off
                state.buf[a0:a0 + cnt].copy_(recv[b][j, :cnt])
            else:
                mover.unpack(lbits, m, pp.sel, off, cnt, recv[b][j])
                launches += 1
        pending = nxt
    return launches
