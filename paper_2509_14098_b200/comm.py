"""Inter-GPU qubit remap: the Pack -> Exchange -> Unpack of executor.py:224-281
when the swapped rank bits select different GPUs.

With one process per GPU, a swap of device-id bit e_i with local bit l_i
(i < m) is a pairwise in-place exchange: process w, whose id reads alpha at
the e bits, trades its region {local l-bits = v} with peer w[e := v] for
every v != alpha, and the peer's data lands in that same region (derivation
in DESIGN.md "Remap").  Two implementations:

* peer memory (default, ``peer_exchange``): the state buffers are allocated
  symmetrically and mapped into every process with CUDA IPC; one bulk-copy
  (TMA-engine) kernel swaps each process's half of every pair over NVLink in
  place, ordered between GPUs by flag words written with stream memory
  operations, optionally chunk by chunk beside the sweeps;
* NCCL (``exchange``, SVB200_REMAP=nccl): regions are packed into staging
  buffers by a CUDA kernel, moved with grouped NCCL send/recv (all 2^m - 1
  peers in one group) and unpacked, double-buffered by chunk.

The data movement of ``exchange`` is injectable so its protocol can be tested
with the gloo backend on CPU tensors (tests/test_comm_gloo.py); the peer
schedule is replayed on CPU in tests/test_peer_schedule.py.
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


# ---------------------------------------------------------------------------
# Peer-memory remap (default on CUDA): symmetric state storage mapped into
# every process with CUDA IPC, one in-place bulk-copy swap kernel per
# exchange (or per chunk of it), ordered between GPUs by flag words that the
# streams write into each other's memory.
# ---------------------------------------------------------------------------

PEER_MODE = os.environ.get("SVB200_REMAP", "peer")  # "peer" | "nccl"
# bulk swap geometry: 148 one-warp CTAs with 3 x 2 x 4 KiB stages (24.7 KB of
# shared memory, 48 registers) fit on every SM beside a running sweep CTA and
# still reach ~690 GB/s per direction (tools/p2p_bench.py, round 1)
SWAP_GRID = int(os.environ.get("SVB200_SWAP_GRID", "0"))  # 0: one CTA per SM
SWAP_PIECE = int(os.environ.get("SVB200_SWAP_PIECE", "4096"))
SWAP_STAGES = int(os.environ.get("SVB200_SWAP_STAGES", "3"))
SWAP_AHEAD = int(os.environ.get("SVB200_SWAP_AHEAD", "1"))

MIN_BULK_RUN = 4096  # contiguous bytes below which the register swap kernel is used

FLAG_RANKS = 64  # flag words: [kind][source rank][chunk], uint32 epochs
FLAG_CHUNKS = 64
FLAG_BYTES = 2 * FLAG_RANKS * FLAG_CHUNKS * 4
READY, DONE = 0, 1


class _Arena:
    """One cudaMalloc'd state buffer (+ flag words) of this process, reusable across runs."""

    def __init__(self, lib, device, nbytes: int):
        import ctypes

        from . import _native

        ptr = ctypes.c_void_p()
        with torch.cuda.device(device):
            _native.check(lib.svb_dev_alloc(nbytes + FLAG_BYTES, ctypes.byref(ptr)), "svb_dev_alloc")
            h = (ctypes.c_uint8 * 64)()
            _native.check(lib.svb_ipc_handle(ptr, h), "svb_ipc_handle")
            flags = torch.as_tensor(_Lease(self, FLAG_BYTES // 4, ptr.value + nbytes, "<i4", hold=False),
                                    device=torch.device("cuda", device))
            flags.zero_()
        self.ptr, self.nbytes, self.device = ptr.value, nbytes, device
        self.handle = bytes(h)
        self.busy = False
        self.epoch = 0  # last flag value used with this buffer
        self.last_use = None  # event after the last GPU work of the previous run on this buffer


class _Lease:
    """Keeps an arena busy while any tensor viewing it is alive."""

    def __init__(self, arena: _Arena, n: int, ptr: int | None = None, typestr: str = "<c16",
                 hold: bool = True):
        self.arena = arena if hold else None
        if hold:
            arena.busy = True
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": typestr, "data": (arena.ptr if ptr is None else ptr, False),
            "version": 2, "strides": None,
        }

    def __del__(self):
        if self.arena is not None:
            self.arena.busy = False


class PeerContext:
    """This process's view of the symmetric state: the peers' mapped state
    and flag pointers and the flag epoch the group agreed on."""

    def __init__(self, me: int, arena: _Arena, peers: dict, peer_flags: dict, epoch: int):
        self.me = me
        self.arena = arena
        self.peers = peers
        self.peer_flags = peer_flags
        self.flags = arena.ptr + arena.nbytes
        self.epoch = epoch
        self.ready = None  # event the buffer's previous run must reach before it is overwritten

    def next_epoch(self) -> int:
        self.epoch += 1
        self.arena.epoch = self.epoch
        return self.epoch

    @staticmethod
    def _off(kind: int, src: int, chunk: int) -> int:
        # the words live in the peers' allocations: an index past the table
        # would write into their state
        if not (0 <= src < FLAG_RANKS and 0 <= chunk < FLAG_CHUNKS and kind in (READY, DONE)):
            raise ValueError(f"flag word out of range (kind {kind}, rank {src}, chunk {chunk}): "
                             f"at most {FLAG_RANKS} processes and {FLAG_CHUNKS} chunks")
        return 4 * ((kind * FLAG_RANKS + src) * FLAG_CHUNKS + chunk)

    def signal(self, kind, chunk, ranks, epoch, stream) -> None:
        """After the stream's earlier work, tell `ranks` that this process reached (kind, chunk)."""
        from . import _native

        lib = _native.load()
        for r in ranks:
            _native.check(lib.svb_stream_write_u32(self.peer_flags[r] + self._off(kind, self.me, chunk),
                                                   epoch, stream), "svb_stream_write_u32")

    def wait(self, kind, chunk, ranks, epoch, stream) -> None:
        """Hold the stream until every rank in `ranks` signalled (kind, chunk) for this epoch."""
        from . import _native

        lib = _native.load()
        for r in ranks:
            _native.check(lib.svb_stream_wait_u32(self.flags + self._off(kind, r, chunk), epoch, stream),
                          "svb_stream_wait_u32")


_ARENAS: dict = {}  # device index -> [_Arena]
_PEER_PTRS: dict = {}  # (device index, peer handle bytes) -> mapped pointer


def release_arenas(group=None) -> int:
    """Free the pooled state buffers no live state uses, and unmap every
    peer buffer.  Collective over `group` (every process calls it); returns
    the number of buffers freed here."""
    import torch.distributed as dist

    from . import _native

    lib = _native.load()
    torch.cuda.synchronize()
    if dist.is_available() and dist.is_initialized():
        dist.barrier(group=group)  # no peer still reads or writes our buffers
    for (di, _), ptr in list(_PEER_PTRS.items()):
        with torch.cuda.device(di):
            _native.check(lib.svb_ipc_close(ptr), "svb_ipc_close")
    _PEER_PTRS.clear()
    freed = 0
    for di, pool in _ARENAS.items():
        keep = []
        for a in pool:
            if a.busy:
                keep.append(a)
                continue
            with torch.cuda.device(di):
                _native.check(lib.svb_dev_free(a.ptr), "svb_dev_free")
            freed += 1
        pool[:] = keep
    if dist.is_available() and dist.is_initialized():
        dist.barrier(group=group)
    return freed


# the IPC-handle exchange of symmetric_buffer runs on a host (gloo) group:
# an NCCL all-gather is ordered after the previous circuit's kernels on the
# stream, and reading it back blocked the host until that circuit finished,
# so a second circuit could not be enqueued while the first ran
HOST_HANDSHAKE = os.environ.get("SVB200_HOST_HANDSHAKE", "1") not in ("0", "false", "no")
_CTRL: dict = {}


def _ctrl_group(group):
    """A gloo group over the whole world for host-side metadata (None: use
    `group` itself).  Only for the default group: new_group is collective
    over every process, which all of them reach here only in that case."""
    import torch.distributed as dist

    if not HOST_HANDSHAKE or group is not None:
        return None
    if dist.get_backend() == "gloo":
        return dist.group.WORLD
    g = _CTRL.get("world")
    if g is None:
        g = _CTRL["world"] = dist.new_group(backend="gloo")
    return g


def symmetric_buffer(n: int, device, group):
    """A complex128 buffer of n amplitudes on `device` in storage every
    process of `group` has mapped; returns (tensor, PeerContext).

    Collective: every process of the group calls it with the same n.  A
    buffer goes back to the pool when the last tensor viewing it dies.
    """
    import ctypes

    import torch.distributed as dist

    from . import _native

    lib = _native.load()
    device = torch.device(device)
    di = device.index if device.index is not None else torch.cuda.current_device()
    nbytes = n * 16
    pool = _ARENAS.setdefault(di, [])
    arena = next((a for a in pool if not a.busy and a.nbytes == nbytes), None)
    if arena is None:
        arena = _Arena(lib, di, nbytes)
        pool.append(arena)
    ready = arena.last_use  # the previous run on this buffer (compute or out= copy) may still use it
    if ready is not None:
        torch.cuda.current_stream(device).wait_event(ready)
        arena.last_use = None
    buf = torch.as_tensor(_Lease(arena, n), device=device)
    me, world = dist.get_rank(group), dist.get_world_size(group)
    if world > FLAG_RANKS:
        raise ValueError(f"peer-memory remap supports at most {FLAG_RANKS} processes (got {world})")
    rec = np.frombuffer(arena.handle + int(arena.epoch).to_bytes(8, "little"), dtype=np.uint8)
    ctrl = _ctrl_group(group)
    mine = torch.from_numpy(rec.copy())
    if ctrl is None:
        mine = mine.to(device)
    allr = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allr, mine, group=ctrl if ctrl is not None else group)
    peers, peer_flags, epoch = {}, {}, 0
    for r, t in enumerate(allr):
        raw_all = bytes(t.cpu().numpy().tobytes())
        epoch = max(epoch, int.from_bytes(raw_all[64:], "little"))
        if r == me:
            continue
        hb = raw_all[:64]
        key = (di, hb)
        if key not in _PEER_PTRS:
            ptr = ctypes.c_void_p()
            raw = (ctypes.c_uint8 * 64).from_buffer_copy(hb)
            with torch.cuda.device(di):
                _native.check(lib.svb_ipc_open(raw, ctypes.byref(ptr)), "svb_ipc_open")
            _PEER_PTRS[key] = ptr.value
        peers[r] = _PEER_PTRS[key]
        peer_flags[r] = peers[r] + nbytes
    ctx = PeerContext(me, arena, peers, peer_flags, epoch)
    ctx.ready = ready
    return buf, ctx


_BARRIER: dict = {}


def device_barrier(group, device) -> None:
    """Stream-ordered barrier: a one-element NCCL all-reduce, so work after
    it starts only once every process has finished the work before it."""
    import torch.distributed as dist

    t = _BARRIER.get(device)
    if t is None:
        t = _BARRIER[device] = torch.zeros(1, dtype=torch.float32, device=device)
    dist.all_reduce(t, group=group)


def swap_args(state, remote: list, me: int, ctx: PeerContext, cbits=None, cval: int = 0):
    """Arguments of svb_peer_swap(_bulk) for one exchange (or its chunk cval
    over `cbits`): process w and peer p = w[e := v] own the pairs
    w.region(v)[k] <-> p.region(alpha_w)[k]; the lower-ranked of the two swaps
    the first half of k, the other the second half."""
    import ctypes

    m = len(remote)
    ebits = [e for e, _ in remote]
    cbits = list(cbits or [])
    k = len(cbits)
    lbits = [lb for _, lb in remote] + cbits
    alpha = 0
    for e in ebits:
        alpha = (alpha << 1) | ((me >> e) & 1)
    # partners in order of sel ^ alpha: round s pairs every process with a
    # distinct partner (a perfect matching), so no process is every partner's first
    plans = sorted(peer_plan(me, ebits, m), key=lambda pp: pp.sel ^ alpha)
    mm = m + k
    region = state.rows << (state.L - mm)
    half = region // 2
    n = len(plans)
    keep = [np.asarray(lbits, dtype=np.int32),
            np.asarray([(pp.sel << k) | cval for pp in plans], dtype=np.uint64),
            np.full(n, (alpha << k) | cval, dtype=np.uint64),
            np.asarray([0 if me < pp.peer else half for pp in plans], dtype=np.int64),
            np.asarray([half if me < pp.peer else region - half for pp in plans], dtype=np.int64)]
    ptrs = (ctypes.c_void_p * n)(*[ctx.peers[pp.peer] for pp in plans])
    from . import _native

    args = (state.buf.data_ptr(), ptrs, n, state.rows, state.L, keep[0].ctypes.data_as(_native._pi32), mm,
            keep[1].ctypes.data, keep[2].ctypes.data, keep[3].ctypes.data, keep[4].ctypes.data)
    return args, [pp.peer for pp in plans], (keep, ptrs)


SWAP_TIMES: list = []  # (start, end) events of every swap kernel, drained by run_plan


def peer_exchange(state, remote: list, ctx: PeerContext, stream, epoch: int, cbits=None, cval: int = 0,
                  wait_done: bool = True) -> int:
    """One exchange (or chunk `cval` of it) as a flag-ordered bulk swap on
    `stream`: signal READY, wait for every partner's READY, swap, signal
    DONE and (wait_done) wait for every partner's DONE -- without it the
    caller must wait_partners_done() before touching the chunk again.
    Returns the kernel launches."""
    from . import _native

    lib = _native.load()
    from .executor import _mark

    args, partners, _keep = swap_args(state, remote, ctx.me, ctx, cbits, cval)
    cur = torch.cuda.current_stream()
    es = cur if cur.cuda_stream == stream else torch.cuda.ExternalStream(stream)
    ts = es if _TRACE_ON() else None
    _mark(f"x{epoch}.{cval} ready-signal", ts)
    ctx.signal(READY, cval, partners, epoch, stream)
    ctx.wait(READY, cval, partners, epoch, stream)
    _mark(f"x{epoch}.{cval} swap start", ts)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(es)
    run = 16 << min([lb for _, lb in remote] + list(cbits or []))  # bytes per contiguous run
    if run >= MIN_BULK_RUN:
        grid = SWAP_GRID or torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        _native.check(lib.svb_peer_swap_bulk(*args, grid, SWAP_PIECE, SWAP_STAGES, SWAP_AHEAD, stream),
                      "svb_peer_swap_bulk")
    else:  # short runs: 16-byte register loads/stores from every SM
        _native.check(lib.svb_peer_swap(*args, 0, 0, stream), "svb_peer_swap")
    e1.record(es)
    SWAP_TIMES.append((e0, e1))
    _mark(f"x{epoch}.{cval} swap end", ts)
    ctx.signal(DONE, cval, partners, epoch, stream)
    if wait_done:
        ctx.wait(DONE, cval, partners, epoch, stream)
        _mark(f"x{epoch}.{cval} done", ts)
    return 1


def wait_partners_done(state, remote: list, ctx: PeerContext, stream, epoch: int, cval: int = 0) -> None:
    """Hold `stream` until every partner of this exchange finished its swap of chunk cval."""
    partners = [pp.peer for pp in peer_plan(ctx.me, [e for e, _ in remote], len(remote))]
    ctx.wait(DONE, cval, partners, epoch, stream)


def _TRACE_ON() -> bool:
    from . import executor

    return executor._TRACE
