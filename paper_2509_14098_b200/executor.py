"""Drop-in replacement for the reference's simulation path.

Mirrors ``svpart/executor.py`` (``run_plan`` :179-307, ``gather`` :320,
``scatter`` :329, ``compare`` :361, ``sample`` :375, ``oracle_simulate``
:346): same names, argument meaning, result types and exceptions.  The
difference is where the state lives and how tasks execute:

* the state is a complex128 CUDA tensor of shape (rows, 2^L); one process per
  GPU holds 2^g / world consecutive ranks as rows (all ranks on one GPU when
  not running distributed);
* every ApplyFused task is compiled once (``program.py``, with a global
  physical-layout planner) and runs as a few fused sweep kernels, generated
  per sweep with NVRTC (``jit.py``) or interpreted for small states
  (``csrc/sweep.cu``);
* Pack -> Exchange -> Unpack is a relabel of layout bits for ranks on the
  same GPU and, between GPUs, an in-place peer-memory swap over NVLink that
  overlaps the sweeps around it (``comm.py``, ``csrc/peer.cu``; NCCL with
  SVB200_REMAP=nccl);
* the norm drift check is accumulated on the device inside the sweep and
  validated once at the end of the run (same exception, same threshold);
* sampling, compare and fidelity run on the device, shard by shard.

There is no CPU execution path: without the CUDA library every call raises.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from . import program as prog
from .errors import DimensionMismatch, NonUnitaryDrift, PlanInvalid, TooLarge

DRIFT_TOL = 1e-8  # executor.py:221


@dataclass
class DistState:
    blocks: torch.Tensor  # (rows on this device, 2^L) complex128, CUDA
    phase: int
    d: int
    g: int
    layouts: list
    rank_base: int = 0  # global rank id of row 0
    world: int = 1
    group: object = None


@dataclass
class RunStats:
    task_counts: dict
    compute_seconds: float
    exchange_seconds: float
    amps_moved: int
    bytes_moved: int
    exchanges: list
    compile_seconds: float = 0.0
    sweeps: int = 0
    kernel_launches: int = 0
    layout_seconds: float = 0.0  # trailing sweeps restoring the reference layout
    swap_seconds: float = 0.0  # inter-GPU swap kernels alone (event-timed, no waits)
    nvlink_bytes: int = 0  # bytes this process sent over NVLink (= received)
    # HBM bytes the sweep launches had to move (16 B per amplitude read or
    # written; sparse sweeps of a |0...0> start move less, prog.sparse_bytes)
    sweep_bytes: int = 0
    # with executor.PROFILE_SWEEPS: descriptor -> [(bytes, ms)] per launch
    sweep_profile: dict = field(default_factory=dict)
    trace: list = field(default_factory=list)  # (label, ms from run start) with SVB200_TRACE=1


@dataclass
class RunResult:
    state: DistState
    histogram: dict | None
    stats: RunStats
    copied: object = None  # CUDA event of the run_plan(out=...) device-to-host copy
    _finish: object = field(default=None, repr=False)  # run_plan(wait=False): deferred end of run

    def wait(self) -> "RunResult":
        """Finish a run_plan(wait=False) run (timings, drift check) and block
        until the out= copy of the final blocks has landed."""
        if self._finish is not None:
            fin, self._finish = self._finish, None
            fin()
        if self.copied is not None:
            self.copied.synchronize()
        return self


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def _arg_device(x):
    """CUDA device of a DistState / tensor argument (None otherwise)."""
    if isinstance(x, DistState):
        x = x.blocks
    if isinstance(x, torch.Tensor) and x.device.type == "cuda":
        return x.device
    return None


def _on_device(pick):
    """Run the wrapped entry point with its CUDA device current: kernels,
    events, torch streams and JIT attributes bind to the current device, so
    a device= argument (or a state on another GPU) must be made current."""
    import functools

    def deco(fn):
        @functools.wraps(fn)
        def wrapper(*args, **kw):
            dev = pick(*args, **kw)
            if dev is None:
                return fn(*args, **kw)
            dev = torch.device(dev)
            if dev.type != "cuda":
                return fn(*args, **kw)
            with torch.cuda.device(dev):
                return fn(*args, **kw)
        return wrapper
    return deco


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _require_cuda(device=None) -> torch.device:
    _native.load()
    if not torch.cuda.is_available():
        raise _native.NativeError("CUDA device required: the B200 executor has no CPU path")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _dist_info(group=None):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


# runs from |0...0> compute only the support of the state until it covers
# the device (program.sparse_start)
SPARSE_START = os.environ.get("SVB200_SPARSE_START", "1") not in ("0", "false", "no")
# runs from |0...0> whose first remap follows only sparse sweeps: every process
# computes that prefix itself and the remap moves no data (program.localize_applies)
LOCALIZE = os.environ.get("SVB200_LOCALIZE", "1") not in ("0", "false", "no")
# generated kernels compile in the background; each launch waits only for its own
PIPELINED_JIT = os.environ.get("SVB200_JIT_PIPELINE", "1") not in ("0", "false", "no")
# sparse sweeps that only expand dead bits are merged into the sweep before (_broadcast_merges)
BROADCAST_MERGE = os.environ.get("SVB200_BROADCAST_MERGE", "1") not in ("0", "false", "no")
# per-launch CUDA events around every sweep (bench.py's roofline); off by default
PROFILE_SWEEPS = False
# self-check mode (SVB200_GUARD_AMPS=n): guard bands of n amplitudes around the
# state, verified when the run finishes (tests/test_selfcheck_gpu.py)
GUARD_AMPS = int(os.environ.get("SVB200_GUARD_AMPS", "0"))
GUARD_VALUE = complex(float("nan"), -7.25)
_prof_log: list | None = None  # (descriptor, bytes, start event, end event) of the current run
JIT_MIN_D = int(os.environ.get("SVB200_JIT_MIN_D", "16"))
# register slots per thread in generated kernels.  4 (256 threads x 16
# amplitudes) needs one shared-memory round trip per 4 dense qubits instead of
# per 3; with the 3-buffer rotation it measured 24.0 vs 27.4 ms on QFT-30 and
# 1.28 vs 1.38 s on QV-30 (B200, round 1)
JIT_REG_BITS = int(os.environ.get("SVB200_JIT_RB", "4"))


def _use_jit(geo: prog.DeviceGeometry, jit) -> bool:
    if jit is not None:
        return bool(jit)
    env = os.environ.get("SVB200_JIT")
    if env is not None:
        return env not in ("0", "false", "no")
    return geo.D >= JIT_MIN_D


@dataclass
class _Compiled:
    blob: torch.Tensor
    descs: np.ndarray
    steps: dict  # task id -> prog.Step; None -> trailing materialization step
    init_perm: list  # reference device bit -> physical bit at Alloc
    n_fused: int
    compile_seconds: float
    host_blob: np.ndarray = field(repr=False, default=None)
    overlap: dict = field(default_factory=dict)  # descriptor -> overlapped exchange step
    cbits: dict = field(default_factory=dict)  # descriptor -> chunk bits its kernel was built with
    kernels: list | None = None  # per-descriptor JIT kernel handles (None: interpreter)
    desc_bytes: list = field(default_factory=list)  # per descriptor: HBM bytes one full launch moves
    norm_alias: dict = field(default_factory=dict)  # slot -> slot whose sweep measured its norm
    dev_index: int = 0
    kernel_names: list = field(default_factory=list)
    kernel_keys: list = field(default_factory=list)  # JIT cache keys (jit._cached) of the cubins
    wait_seconds: float = 0.0  # host time blocked on kernels still compiling (pipelined JIT)
    jit_seconds: float = 0.0
    zero_init: dict = field(default_factory=dict)  # descriptors that synthesise |0...0>
    sparse: dict = field(default_factory=dict)  # descriptor -> (support, full_out), prog.sparse_start
    skip: set = field(default_factory=set)  # descriptors merged into the sweep before (_broadcast_merges)
    bcast: dict = field(default_factory=dict)  # descriptor -> broadcast store (_broadcast_merges)
    n_sweeps: int = 0


_compile_cache: dict = {}


def compile_plan(plan, geo: prog.DeviceGeometry, device, jit=None, zero_start: bool = False) -> _Compiled:
    """Compile every ApplyFused task of the plan for this device (cached).

    zero_start: the run starts from |0...0>, so the first sweep (if no remap
    precedes it) synthesises its tiles instead of reading a zeroed state."""
    import time

    use_jit = _use_jit(geo, jit)
    key = (id(plan), len(plan.tasks), geo.d, geo.g, geo.h, geo.rank_base, str(device), use_jit,
           zero_start, SPARSE_START)
    hit = _compile_cache.get(key)
    if hit is not None and hit[0] is plan:
        return hit[1]
    t0 = time.perf_counter()
    dist_run = _dist_info()[1] > 1
    ob = _overlap_bits() if (use_jit and dist_run) else 0
    skip_first = replicate = False
    world = _dist_info()[1]
    if use_jit and zero_start and SPARSE_START and world > 1:
        dp0 = prog.plan_device(plan, geo, rb=JIT_REG_BITS, overlap_bits=0, free_start=True,
                               stable_threads=jitmod_shuffle())
        skip_first = prog.sparse_reaches_first_remap(dp0, geo.D)
        replicate = LOCALIZE and prog.localize_applies(dp0, geo.D, world, geo.h)
    dp = prog.plan_device(plan, geo, rb=JIT_REG_BITS if use_jit else prog.RB, overlap_bits=ob,
                          free_start=zero_start, stable_threads=use_jit and jitmod_shuffle(),
                          overlap_skip_first=skip_first, replicate_prefix=replicate)
    blob, descs, _ = prog.pack(dp.buf)
    host = np.ascontiguousarray(blob)
    dev_blob = torch.from_numpy(host).to(device)
    steps = {}
    for st in dp.steps:
        steps[st.task_id] = st
    # sweeps launched in parts around an overlapped remap: descriptor ->
    # {"pre": exchange it feeds, "post": exchange it waits for,
    #  "chain": exchange whose depth-first chain starts here}
    overlap = {}
    for st in dp.steps:
        if st.kind == "exchange" and st.cbits and all(ib >= geo.h for ib, _ in st.swaps):
            overlap.setdefault(st.pre, {})["pre"] = st
            overlap.setdefault(st.post, {})["post"] = st
            overlap.setdefault(st.chain[0], {})["chain"] = st
    out = _Compiled(dev_blob, descs, steps, dp.init_perm, dp.n_fused, time.perf_counter() - t0,
                    host, n_sweeps=len(dp.buf.descs))
    out.norm_alias = dict(dp.norm_alias)
    out.overlap = overlap if use_jit else {}
    out.cbits = {i: d["cbits"] for i, d in enumerate(dp.buf.descs) if d.get("cbits")} if use_jit else {}
    if use_jit and dp.buf.descs:
        from . import jit as jitmod

        t1 = time.perf_counter()
        unit = geo.rank_base == 0 or any(st.kind == "localize" for st in dp.steps)  # replicas hold it too
        sparse = prog.sparse_start(dp, geo.D, unit) if (zero_start and SPARSE_START) else {}
        ld_xor = _fold_localize(dp, geo, sparse)
        st_keep = _prefix_store_masks(dp, geo, sparse)
        out.st_keep = st_keep
        bcast = _broadcast_merges(dp, geo, sparse, ld_xor, st_keep, overlap) if BROADCAST_MERGE else {}
        out.skip = {j + 1 for j in bcast}
        for j, (_, _, _, slot_j) in bcast.items():
            descs[j]["norm_slot"] = slot_j
        out.bcast = bcast
        names, slots = jitmod.build_kernels(dp.buf, sparse=sparse, lazy=PIPELINED_JIT, ld_xor=ld_xor,
                                            st_keep=st_keep, bcast=bcast, skip=out.skip)
        out.zero_init = dict(jitmod._LAST_ZERO_INIT)
        out.sparse = sparse
        for i, gcount in jitmod._LAST_GROUPS.items():  # launch geometry of two-group kernels
            descs[i]["groups"] = gcount
        dev_index = device.index if device.index is not None else torch.cuda.current_device()
        out.dev_index = dev_index
        out.kernel_names = list(names)
        if PIPELINED_JIT:  # resolved at first launch (_kernel): early sweeps run while later ones compile
            out.kernels = list(slots)
            out.kernel_keys = [sl.h if sl is not None else None for sl in slots]
        else:
            out.kernels = [jitmod.load_kernel(n, c, dev_index) if n is not None else None
                           for n, c in zip(names, slots)]
        out.jit_seconds = time.perf_counter() - t1
    keep = getattr(out, "st_keep", {})
    bc = getattr(out, "bcast", {})

    def launch_bytes(i, d):
        if i in out.skip:
            return 0
        rd, wr = prog.sparse_bytes(d, out.sparse.get(i))
        if i in keep:  # a store mask writes one region of the masked bits
            wr >>= bin(keep[i][0]).count("1")
        if i in bc:  # broadcast stores: every value to 2^|F| positions
            wr <<= bin(bc[i][0]).count("1")
        return rd + wr

    out.desc_bytes = [launch_bytes(i, d) for i, d in enumerate(dp.buf.descs)]
    _compile_cache.clear()  # keep one plan resident
    _compile_cache[key] = (plan, out)
    return out


def jitmod_shuffle() -> bool:
    """Planner-chosen stable thread-bit orders (warp-local stage changes)."""
    from . import jit as jitmod

    return jitmod.SHUFFLE_STAGES or jitmod.LOCAL_STAGES


def _has_remote(st, geo) -> bool:
    return any(ib >= geo.h for ib, _ in st.swaps)


def _storage_bitperm(layout, d: int, to_basis: bool) -> list:
    """Bit map of _storage_to_basis (executor.py:310-317), LSB-indexed."""
    perm = [0] * d
    for q in range(d):
        s_bit = d - 1 - layout[q]
        b_bit = d - 1 - q
        if to_basis:
            perm[s_bit] = b_bit
        else:
            perm[b_bit] = s_bit
    return perm


def _bitperm(src: torch.Tensor, dst: torch.Tensor, perm: list) -> None:
    lib = _native.load()
    arr, p32 = _native.i32_array(perm)
    _native.check(
        lib.svb_bitperm(src.data_ptr(), dst.data_ptr(), len(perm), p32, _stream_ptr(src.device)),
        "svb_bitperm",
    )


def _two_involutions(perm: list) -> tuple[list, list]:
    """Write a bit permutation (bit r -> perm[r]) as b(a(r)) with a, b
    involutions: lists of disjoint transpositions, one in-place bitswap each."""
    n = len(perm)
    seen = [False] * n
    a, b = [], []
    for start in range(n):
        if seen[start]:
            continue
        cyc = [start]
        seen[start] = True
        while not seen[perm[cyc[-1]]]:
            cyc.append(perm[cyc[-1]])
            seen[cyc[-1]] = True
        k = len(cyc)
        if k < 2:
            continue
        # a: c_i <-> c_{-i}, b: c_i <-> c_{1-i} (indices mod k), so b(a(c_i)) = c_{i+1}
        for i in range(k):
            j = (-i) % k
            if i < j:
                a.append((cyc[i], cyc[j]))
            j = (1 - i) % k
            if i < j:
                b.append((cyc[i], cyc[j]))
    return a, b


def _bitswap_pass(state, D: int, pairs: list, stream) -> None:
    """Disjoint transpositions commute: apply them 8 per svb_bitswap launch."""
    lib = _native.load()
    for i in range(0, len(pairs), 8):
        grp = pairs[i:i + 8]
        u = np.asarray([x for x, _ in grp], dtype=np.int32)
        w = np.asarray([y for _, y in grp], dtype=np.int32)
        _native.check(lib.svb_bitswap(state.buf.data_ptr(), D, u.ctypes.data_as(_native._pi32),
                                      w.ctypes.data_as(_native._pi32), len(grp), stream), "svb_bitswap")


def _initial_blocks(initial, plan, rank_base: int, rows: int, world: int):
    """This process's rank blocks (rows, 2^L) of `initial` at layout phase 0,
    in the reference storage order (executor.py:329-343)."""
    d, g = plan.d, plan.g
    L = d - g
    if isinstance(initial, DistState):
        if initial.phase != 0:
            raise PlanInvalid(f"initial state is at layout phase {initial.phase}, run_plan starts at 0")
        initial = initial.blocks
    t = initial if isinstance(initial, torch.Tensor) else torch.from_numpy(np.asarray(initial))
    if t.dtype != torch.complex128:
        t = t.to(torch.complex128)
    if t.dim() == 2:
        if tuple(t.shape) == (rows, 1 << L):
            return t
        if tuple(t.shape) == (1 << g, 1 << L):
            return t[rank_base:rank_base + rows]
        raise DimensionMismatch(f"initial blocks {tuple(t.shape)} != ({rows}, 2^{L}) or (2^{g}, 2^{L})")
    if tuple(t.shape) != (1 << d,):
        raise DimensionMismatch(f"state length {tuple(t.shape)} != 2^{d}")
    # dense basis vector (qubit 0 = MSB): view it with one axis per qubit, order
    # the axes by storage position, fix this process's top rank bits, and copy
    # only its 2^(L+h) amplitudes
    layout = plan.layout_phases[0]
    q_of_pos = [0] * d
    for q, pos in enumerate(layout):
        q_of_pos[pos] = q
    x = t.reshape((2,) * d).permute(q_of_pos) if d else t
    h = rows.bit_length() - 1
    top = g - h
    for i in range(top):
        x = x[(rank_base >> (g - 1 - i)) & 1]
    return x.reshape(rows, 1 << L)


def _load_initial(state, initial, plan, rank_base, rows, world, device, local_perm) -> None:
    """Copy this process's share of `initial` into the state and move its
    local bits to the planner's initial physical layout in place."""
    blocks = _initial_blocks(initial, plan, rank_base, rows, world)
    if blocks.device.type == "cpu" and blocks.is_pinned():
        # upload on its own stream: it can then run beside an earlier run's
        # out= download (full-duplex PCIe) and an earlier run's compute
        up = _upload_stream(device)
        cur = torch.cuda.current_stream(device)
        if state.upload_stream is not up and state.ctx is None:
            up.wait_stream(cur)  # the buffer may still be in use by work on `cur`
        if state.ctx is not None and state.ctx.ready is not None:
            up.wait_event(state.ctx.ready)  # a pooled peer buffer's previous run
        with torch.cuda.stream(up):
            state.blocks.copy_(blocks, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(up)
        cur.wait_event(ev)
        if state.upload_stream is not up:
            state.buf.record_stream(up)
    else:
        state.blocks.copy_(blocks, non_blocking=blocks.device.type != "cpu")
    L = state.L
    perm = [int(p) for p in local_perm]
    if perm == list(range(L)):
        return
    D = L + (rows.bit_length() - 1)
    if (rows << L) < prog.NREG:
        D = max(D, 4)
    a, b = _two_involutions(perm)
    stream = _stream_ptr(device)
    _bitswap_pass(state, D, a, stream)
    _bitswap_pass(state, D, b, stream)


class _Flat:
    """The state as one row of L + log2(rows) bits: the planner may keep a
    local qubit on a row bit (and a rank bit on a local one), so remote swaps
    address the whole device index.  Region enumeration is unchanged: rows
    are simply the top free bits."""

    def __init__(self, state):
        self.buf, self.ctx = state.buf, state.ctx
        self.rows = 1
        self.L = state.L + (state.rows.bit_length() - 1)


class _State:
    """Device storage with a phantom pad so tiny states still fill 16 amplitudes."""

    def __init__(self, rows: int, L: int, device, zero: bool = True, group=None, peer: bool = False,
                 upload_stream=None):
        self.rows, self.L = rows, L
        n = rows << L
        self.ctx = None  # comm.PeerContext of the peer-memory remap
        self.upload_stream = None  # set when the buffer was allocated for an upload on that stream
        if peer:
            from . import comm

            self.buf, self.ctx = comm.symmetric_buffer(max(n, prog.NREG), device, group)
            if zero:
                self.buf.zero_()
        elif upload_stream is not None and not zero:
            # allocated on the upload stream: the caching allocator then only
            # hands out memory whose earlier users were uploads, so the upload
            # needs no wait on the compute stream (whose previous circuit may
            # still be running); the compute stream's use is recorded
            with torch.cuda.stream(upload_stream):
                self.buf = torch.empty(max(n, prog.NREG), dtype=torch.complex128, device=device)
            self.buf.record_stream(torch.cuda.current_stream(device))
            self.upload_stream = upload_stream
        elif GUARD_AMPS:
            # self-check mode: the state sits between two guard bands filled
            # with a NaN pattern that run_plan verifies at the end of the run
            m = max(n, prog.NREG)
            self.guarded = torch.empty(m + 2 * GUARD_AMPS, dtype=torch.complex128, device=device)
            self.guarded[:GUARD_AMPS].fill_(GUARD_VALUE)
            self.guarded[GUARD_AMPS + m:].fill_(GUARD_VALUE)
            self.buf = self.guarded[GUARD_AMPS:GUARD_AMPS + m]
            if zero:
                self.buf.zero_()
        else:
            alloc = torch.zeros if zero else torch.empty
            self.buf = alloc(max(n, prog.NREG), dtype=torch.complex128, device=device)
        self.blocks = self.buf[:n].view(rows, 1 << L)

    def check_guards(self) -> None:
        g = getattr(self, "guarded", None)
        if g is None:
            return
        bands = torch.cat([g[:GUARD_AMPS], g[-GUARD_AMPS:]])
        ok = torch.view_as_real(bands).view(torch.int64) == torch.view_as_real(
            torch.full_like(bands, GUARD_VALUE)).view(torch.int64)
        if not bool(ok.all()):
            raise _native.NativeError("guard band around the state was overwritten (out-of-bounds write)")


def _upload_stream(device):
    up = _UPLOAD_STREAMS.get(device)
    if up is None:
        up = _side_stream(_UPLOAD_STREAMS, device)
    return up


def _pinned_host(x) -> bool:
    if isinstance(x, DistState):
        x = x.blocks
    return isinstance(x, torch.Tensor) and x.device.type == "cpu" and x.dim() == 2 and x.is_pinned()


# ---------------------------------------------------------------------------
# run_plan
# ---------------------------------------------------------------------------


_COPY_STREAMS: dict = {}  # device -> stream of run_plan(out=...) downloads
_COMM_STREAMS: dict = {}  # device -> stream of overlapped remap chunks


def _side_stream(cache: dict, device) -> torch.cuda.Stream:
    """A dedicated stream per device and purpose, created once: torch's
    pooled streams (torch.cuda.Stream()) are handed out round-robin from 32
    per device, so a fresh one per run would eventually alias the upload,
    copy or NCCL stream and serialise behind it.  Native handles never alias."""
    st = cache.get(device)
    if st is None:
        from . import _native
        import ctypes

        lib = _native.load()
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            _native.check(lib.svb_stream_create(ctypes.byref(h)), "svb_stream_create")
        st = cache[device] = torch.cuda.ExternalStream(h.value, device=device)
    return st
_UPLOAD_STREAMS: dict = {}  # device -> stream of pinned initial-state uploads
_FENCE: dict = {}  # device -> one-element tensor (see run_plan(out=...))
_META_STREAMS: dict = {}  # device -> stream of the deferred drift-check read (run_plan(wait=False))
_PINNED_POOL: list = []  # pinned float64 readback buffers, returned by each run's finish()


def _pinned_take(n: int) -> torch.Tensor:
    for i, t in enumerate(_PINNED_POOL):
        if t.numel() >= n:
            return _PINNED_POOL.pop(i)
    return torch.empty(max(n, 4096), dtype=torch.float64, pin_memory=True)


@_on_device(lambda plan, *a, device=None, **k: device)
def run_plan(plan, shots: int | None = None, seed: int | None = None, initial=None, *,
             device=None, group=None, grid_limit: int = 0, jit=None, out=None,
             wait: bool = True) -> RunResult:
    """Interpret the task list on the GPU(s); returns the final state and optional histogram.

    Same contract as ``svpart.executor.run_plan`` (executor.py:179-307).
    Under ``torch.distributed`` every process holds ``2^g / world`` ranks.

    out: optional host tensor (pinned for asynchrony) of this process's
    rows x 2^L amplitudes.  The final blocks are copied into it on a copy
    stream and run_plan returns without waiting (``result.wait()`` does), so
    one circuit's download overlaps the next circuit's upload.

    wait=False: return as soon as every kernel and copy is enqueued;
    ``result.wait()`` then finishes the run (event timings, the drift check,
    which raises NonUnitaryDrift there, and the out= copy), so the next
    circuit's upload can overlap this one's compute as well.
    """
    device = _require_cuda(device)
    lib = _native.load()
    d, g = plan.d, plan.g
    L = d - g
    me, world = _dist_info(group)
    nranks = 1 << g
    if world > nranks or nranks % world:
        raise PlanInvalid(f"{nranks} ranks cannot be split over {world} processes")
    rows = nranks // world
    h = rows.bit_length() - 1
    rank_base = me * rows
    geo = prog.DeviceGeometry(d=d, g=g, h=h, rank_base=rank_base)
    # tiny states are padded with zero phantom bits up to one 16-amplitude tile
    geo_eff = prog.DeviceGeometry(d=d, g=g, h=h, rank_base=rank_base, pad_to=prog.RB)
    rows_eff = 1 << (geo_eff.D - L)
    stream = _stream_ptr(device)

    stats = RunStats(task_counts={}, compute_seconds=0.0, exchange_seconds=0.0,
                     amps_moved=0, bytes_moved=0, exchanges=[])
    global _prof_log
    prof_log = _prof_log = [] if PROFILE_SWEEPS else None

    # protocol validation happens in task order, like the reference
    state: _State | None = None
    packed = None
    done: set = set()
    compiled = None
    norms = None
    events = []  # (kind, start, end)
    # overlapped remaps: per-chunk events and flag epochs, comm stream, chained sweeps already run
    ovl = {"pre": {}, "unpack": {}, "comm": None, "peer": {}, "launched": set()}
    fused_order = []  # task ids of executed ApplyFused, in order

    def fail(exc):
        # report an earlier drift first, as the reference would have raised it
        _check_norms()
        raise exc

    def _check_norms(vals=None):
        if norms is None or not fused_order:
            return
        if vals is None:
            vals = norms.cpu().numpy()
            if world > 1:
                t = torch.from_numpy(vals).to(device)
                import torch.distributed as dist

                dist.all_reduce(t, group=group)
                vals = t.cpu().numpy()
        for slot, tid in enumerate(fused_order):
            nv = float(vals[compiled.norm_alias.get(slot, slot)])
            if abs(nv - 1.0) > DRIFT_TOL:
                raise NonUnitaryDrift(f"norm drifted to {nv!r}")

    for task in plan.tasks:
        if any(dep not in done for dep in task.deps):
            fail(PlanInvalid(f"task {task.id} runs before its dependencies"))
        kind = task.kind
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        if kind == "Alloc":
            if state is not None:
                fail(PlanInvalid("double Alloc"))
            if task.payload["num_ranks"] != nranks or task.payload["block_len"] != 1 << L:
                fail(PlanInvalid("Alloc payload disagrees with plan shape"))
            compiled = compile_plan(plan, geo_eff, device, jit, zero_start=initial is None)
            stats.compile_seconds = compiled.compile_seconds + compiled.jit_seconds
            wait0 = compiled.wait_seconds
            # when the first sweep synthesises |0...0> the state needs no memset
            from . import comm

            # a memset is needed only when nothing else writes every amplitude:
            # no |0...0>-synthesising first sweep and no initial state (tiny
            # states also keep their phantom pad zero)
            zero = (initial is None and not compiled.zero_init) or (rows << L) < prog.NREG
            state = _State(rows, L, device, zero=zero, group=group,
                           peer=world > 1 and comm.PEER_MODE == "peer",
                           upload_stream=_upload_stream(device) if _pinned_host(initial) else None)
            if initial is None:
                if rank_base == 0 and not compiled.zero_init:
                    state.blocks[0, 0] = 1.0  # |0...0> sits at index 0 in every layout
            else:
                try:
                    _load_initial(state, initial, plan, rank_base, rows, world, device,
                                  compiled.init_perm[:L])
                except (DimensionMismatch, PlanInvalid) as exc:
                    fail(exc)
            # even length: the deferred drift check reads it back in 16-byte units
            norms = torch.zeros(max(compiled.n_fused, 1) + (max(compiled.n_fused, 1) & 1), dtype=torch.float64,
                                device=device)
        elif kind == "ApplyFused":
            if state is None:
                fail(PlanInvalid("compute before Alloc"))
            st = compiled.steps[task.id]
            slot = len(fused_order)
            launched = 0
            if st.count and compiled.overlap:
                launched = _run_descs_overlapped(compiled, st, state, rows_eff, L, norms, grid_limit, stream,
                                                 ovl)
            elif st.count:
                _mark(f"sweeps{st.first}-{st.first + st.count - 1} start")
                launched = _run_descs(compiled, st.first, st.count, state, rows_eff, L, norms, grid_limit,
                                      stream, skip=compiled.skip)
                _mark(f"sweeps{st.first}-{st.first + st.count - 1} end")
            elif slot in compiled.norm_alias:  # merged into a sweep of another leaf
                pass
            elif slot > 0:  # relabel-only leaf: the state (and its norm) is unchanged
                norms[slot:slot + 1].copy_(norms[slot - 1:slot])
            elif initial is None:  # |0...0> (possibly not materialised yet) has norm 1
                norms[0:1].fill_(1.0 / world)
            else:
                lib.svb_norm2(state.buf.data_ptr(), rows << L, norms[slot:].data_ptr(), stream)
                launched = 1
            stats.sweeps += st.count - sum(1 for di in range(st.first, st.first + st.count) if di in compiled.skip)
            stats.sweep_bytes += sum(compiled.desc_bytes[st.first:st.first + st.count])
            stats.kernel_launches += launched
            fused_order.append(task.id)
        elif kind == "Pack":
            if state is None:
                fail(PlanInvalid("Pack before Alloc"))
            if packed is not None:
                fail(PlanInvalid("Pack while a previous Pack is pending"))
            packed = {"phase": task.payload["phase"], "swaps": task.payload["swaps"], "sent": False}
        elif kind == "Exchange":
            if packed is None or packed["swaps"] != task.payload["swaps"]:
                fail(PlanInvalid("Exchange without matching Pack"))
            swaps = task.payload["swaps"]
            m = len(swaps)
            xst = compiled.steps[task.id]
            if xst.kind == "localize":
                launches = _localize(state, xst, geo, stream)
            elif compiled.overlap.get(xst.pre, {}).get("pre") is xst:
                launches, ce0, ce1 = _remap_overlapped(state, xst, geo, group, ovl)
                events.append(("Exchange", ce0, ce1))
            else:
                _mark(f"remap{task.id} start")
                launches = _remap(state, xst.swaps, geo, group, stream)
                _mark(f"remap{task.id} end")
            stats.kernel_launches += launches
            moved = nranks * ((1 << m) - 1) * (1 << (L - m))
            messages = nranks * ((1 << m) - 1)
            mr = sum(1 for ib, _ in xst.swaps if ib >= geo.h)  # swapped bits that cross GPUs
            if mr and xst.kind != "localize":  # this process's bytes over NVLink (sent = received)
                stats.nvlink_bytes += 16 * rows * ((1 << mr) - 1) * (1 << (L - mr))
            packed["sent"] = True
            stats.amps_moved += moved
            stats.bytes_moved += moved * 16
            stats.exchanges.append({"amps": moved, "bytes": moved * 16, "messages": messages})
        elif kind == "Unpack":
            if packed is None or not packed.get("sent"):
                fail(PlanInvalid("Unpack without a completed Exchange"))
            packed = None
        elif kind == "Free":
            if packed is not None:
                fail(PlanInvalid("Free with undelivered messages"))
        else:
            fail(PlanInvalid(f"unknown task kind {kind!r}"))
        ev1.record()
        events.append((kind, ev0, ev1))
        stats.task_counts[kind] = stats.task_counts.get(kind, 0) + 1
        done.add(task.id)

    if state is None:
        raise PlanInvalid("plan never allocated state")
    mat = compiled.steps.get(None)
    if mat is not None and compiled.kernels is not None:  # materialisation kernels, before the clock stops
        for di in range(mat.first, mat.first + mat.count):
            _kernel(compiled, di)
    stats.compile_seconds += compiled.wait_seconds - wait0  # launches that waited for their kernel
    if mat is not None:  # restore the reference layout
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launched = _run_descs(compiled, mat.first, mat.count, state, rows_eff, L, None, grid_limit, stream)
        e1.record()
        events.append(("Materialize", e0, e1))
        stats.sweeps += mat.count
        stats.sweep_bytes += sum(compiled.desc_bytes[mat.first:mat.first + mat.count])
        stats.kernel_launches += launched
    fin_ev = torch.cuda.Event()
    fin_ev.record()
    from . import comm

    swap_events = list(comm.SWAP_TIMES)  # this run's swaps (another run may start before it finishes)
    comm.SWAP_TIMES.clear()
    norm_host = norm_ev = None
    if not wait and norms is not None and fused_order:
        # deferred drift check: reduce on the device now, read back on a side
        # stream, so no small copy ever queues on this stream behind a download
        nsum = norms
        if world > 1:
            import torch.distributed as dist

            nsum = norms.clone()
            dist.all_reduce(nsum, group=group)
        src_ev = torch.cuda.Event()
        src_ev.record()
        ms = _META_STREAMS.get(device)
        if ms is None:
            ms = _side_stream(_META_STREAMS, device)
        ms.wait_event(src_ev)
        norm_host = _pinned_take(nsum.numel())  # pooled: a fresh pinned allocation syncs the device
        with torch.cuda.stream(ms):
            # an SM copy straight into mapped pinned memory: a copy-engine
            # transfer would queue behind the out= downloads of this and the
            # next circuit (measured, tools/pipeline_probe.py)
            _native.check(lib.svb_copy(norm_host.data_ptr(), nsum.data_ptr(), nsum.numel() // 2, 1, ms.cuda_stream),
                          "svb_copy")
            norm_ev = torch.cuda.Event()
            norm_ev.record(ms)
        nsum.record_stream(ms)

    def finish():
        """Host side of the end of the run: event timings and the drift check."""
        fin_ev.synchronize()
        state.check_guards()
        if _TRACE and _marks:
            t0 = _marks[0][1]
            stats.trace = [(lab, t0.elapsed_time(ev)) for lab, ev in _marks]
            _marks.clear()
        for kind, e0, e1 in events:
            sec = e0.elapsed_time(e1) / 1e3
            if kind in ("Pack", "Exchange", "Unpack"):
                stats.exchange_seconds += sec
            elif kind == "ApplyFused":
                stats.compute_seconds += sec
            elif kind == "Materialize":
                stats.layout_seconds += sec
        for e0, e1 in swap_events:
            stats.swap_seconds += e0.elapsed_time(e1) / 1e3
        for di, nb, e0, e1 in prof_log or ():
            stats.sweep_profile.setdefault(di, []).append((nb, e0.elapsed_time(e1)))
        if norm_ev is not None:
            norm_ev.synchronize()
            vals = norm_host.numpy().copy()
            _PINNED_POOL.append(norm_host)
            _check_norms(vals)
        else:
            _check_norms()

    dstate = DistState(
        blocks=state.blocks, phase=len(plan.layout_phases) - 1, d=d, g=g,
        layouts=[list(p) for p in plan.layout_phases], rank_base=rank_base, world=world,
        group=group,
    )
    if not wait and shots is not None:
        raise ValueError("run_plan(shots=...) needs wait=True")
    if wait:
        finish()  # small device-to-host reads go before the big out= copy, not behind it
    histogram = None
    if shots is not None:  # on the device, shard by shard (no gather)
        from . import sampling

        histogram = sampling.sample_state(dstate, shots, seed)
    copied = None
    if out is not None:
        if tuple(out.shape) not in ((rows, 1 << L), (rows << L,)) or out.dtype != torch.complex128:
            raise DimensionMismatch(f"out {tuple(out.shape)} {out.dtype} != ({rows}, 2^{L}) complex128")
        cs = _COPY_STREAMS.get(device)
        if cs is None:
            cs = _side_stream(_COPY_STREAMS, device)
        # The drift check's small device-to-host read was the last operation on
        # this stream; the stream's next operation would then wait behind the
        # download below in the copy-engine queue (measured, tools/copy_overlap.py).
        # A one-element kernel in between keeps the next run's upload free to run.
        fence = _FENCE.get(device)
        if fence is None:
            fence = _FENCE[device] = torch.zeros(1, dtype=torch.int32, device=device)
        fence.zero_()
        cs.wait_event(fin_ev)
        with torch.cuda.stream(cs):
            out.view(rows, 1 << L).copy_(state.blocks, non_blocking=True)
            copied = torch.cuda.Event()
            copied.record(cs)
        state.buf.record_stream(cs)  # the allocator keeps the buffer until the copy is done
    if state.ctx is not None:  # a pooled peer buffer's next user waits for this run's last use
        state.ctx.arena.last_use = copied if copied is not None else fin_ev
    res = RunResult(state=dstate, histogram=histogram, stats=stats, copied=copied)
    if not wait:
        res._finish = finish
    return res


_TRACE = os.environ.get("SVB200_TRACE") == "1"
_marks: list = []


def _mark(label: str, stream=None) -> None:
    """Record a timing event on `stream` (tracing only)."""
    if _TRACE:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        _marks.append((label, ev))


def _overlap_bits() -> int:
    """Chunk bits of remaps that overlap the sweeps around them.  On with the
    peer-memory remap (its bulk-copy swap shares the SMs with the sweeps);
    off with NCCL, whose kernels starve the persistent sweeps (round 1)."""
    from . import comm

    env = os.environ.get("SVB200_OVERLAP_BITS")
    bits = int(env) if env is not None else (3 if comm.PEER_MODE == "peer" else 0)
    if (1 << bits) > comm.FLAG_CHUNKS:  # one flag word per chunk and partner
        raise ValueError(f"SVB200_OVERLAP_BITS={bits}: at most {comm.FLAG_CHUNKS.bit_length() - 1} chunk bits")
    return bits


OVERLAP_GRID = int(os.environ.get("SVB200_OVERLAP_GRID", "0"))  # 0: every SM


def _part_values(cbits, c, fbits):
    """Device-bit and tile-index encodings of chunk value c (cbits[0] = MSB)."""
    k = len(cbits)
    val = tid = 0
    fpos = {b: i for i, b in enumerate(fbits)}
    for j, b in enumerate(cbits):
        if (c >> (k - 1 - j)) & 1:
            val |= 1 << b
            tid |= 1 << fpos[b]
    return val, tid


def _launch_part(compiled, di, state, norms, grid_limit, stream, cbits, c) -> None:
    lib = _native.load()
    d = compiled.descs[di]
    K, D = int(d["K"]), int(d["D"])
    tin = set(int(x) for x in d["tin"][:K])
    fbits = [b for b in range(D) if b not in tin]
    val, tid = _part_values(cbits, c, fbits)
    ntiles = 1 << (D - K - len(cbits))
    ev = _prof_begin()
    rc = lib.svb_jit_launch_sweep_part(_kernel(compiled, di), state.buf.data_ptr(), compiled.blob.data_ptr(),
                                       compiled.descs[di:di + 1].ctypes.data,
                                       norms.data_ptr() if norms is not None else None,
                                       grid_limit, val, tid, ntiles, stream)
    _native.check(rc, "svb_jit_launch_sweep_part")
    _prof_end(ev, di, compiled.desc_bytes[di] >> len(cbits) if compiled.desc_bytes else 0)


def _run_descs_overlapped(compiled, st, state, rows_eff, L, norms, grid_limit, stream, ovl) -> int:
    """Sweeps of one ApplyFused task when remaps overlap the sweeps around
    them.  A sweep next to an overlapped remap runs in parts, one per chunk;
    the chain of sweeps before a remap runs depth-first (chunk c of every
    chain sweep, then an event that lets the remap of chunk c start on the
    comm stream), and part c of the sweep after it waits for that chunk."""
    from . import comm

    grid = min(grid_limit or prog_sms(), OVERLAP_GRID or prog_sms())
    cur = torch.cuda.current_stream()
    launches = 0
    for di in range(st.first, st.first + st.count):
        if di in ovl["launched"]:
            continue  # ran earlier as part of a depth-first chain
        roles = compiled.overlap.get(di)
        if not roles:
            _mark(f"sweep{di} start")
            launches += _run_descs(compiled, di, 1, state, rows_eff, L, norms, grid_limit, stream,
                                   skip=compiled.skip)
            _mark(f"sweep{di} end")
            continue
        group = roles["chain"].chain if "chain" in roles else [di]
        ovl["launched"].update(group)
        cbits = compiled.cbits[di]  # the planner gives a chain and its remap's post the same bits
        for c in range(1 << len(cbits)):
            for dj in group:
                r = compiled.overlap.get(dj, {})
                waits, feeds = r.get("post"), r.get("pre")
                if waits is not None:  # part c needs chunk c of the previous remap ...
                    cur.wait_event(ovl["unpack"][id(waits)][c])
                    if state.ctx is not None:  # ... swapped on both sides of every pair
                        remote, epoch = ovl["peer"][(id(waits), c)]
                        comm.wait_partners_done(state, remote, state.ctx, cur.cuda_stream, epoch, c)
                _mark(f"sweep{dj}.part{c} start", cur)
                _launch_part(compiled, dj, state, norms, grid, stream, cbits, c)
                launches += 1
                _mark(f"sweep{dj}.part{c} end", cur)
                if feeds is not None:
                    ev = torch.cuda.Event()
                    ev.record(cur)
                    ovl["pre"].setdefault(id(feeds), []).append(ev)
    return launches


def prog_sms() -> int:
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def _remap_overlapped(state, xst, geo, group, ovl):
    """Chunked remap on a side stream: chunk c starts when part c of the sweep
    before has been written and releases part c of the sweep after."""
    from . import comm

    if ovl["comm"] is None:
        ovl["comm"] = _side_stream(_COMM_STREAMS, torch.device("cuda", torch.cuda.current_device()))
    cs = ovl["comm"]
    remote = [(ib - geo.h, lb) for ib, lb in xst.swaps]
    pre_evs = ovl["pre"].pop(id(xst))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    outs = []
    epoch = state.ctx.next_epoch() if state.ctx is not None else 0
    with torch.cuda.stream(cs):
        cs.wait_event(pre_evs[0])
        e0.record(cs)
        for c, ev in enumerate(pre_evs):
            cs.wait_event(ev)
            if state.ctx is not None:
                launches += comm.peer_exchange(_Flat(state), remote, state.ctx, cs.cuda_stream, epoch,
                                               cbits=xst.cbits, cval=c, wait_done=False)
                ovl["peer"][(id(xst), c)] = (remote, epoch)
            else:
                launches += comm.exchange(_Flat(state), remote, geo, group, cbits=xst.cbits, cval=c)
            done = torch.cuda.Event()
            done.record(cs)
            outs.append(done)
        e1.record(cs)
    ovl["unpack"][id(xst)] = outs
    return launches, e0, e1


def _kernel(compiled, di: int) -> int:
    """Kernel handle of descriptor di, waiting for its compile if needed."""
    k = compiled.kernels[di]
    if isinstance(k, int):
        return k
    import time

    from . import jit as jitmod

    t0 = time.perf_counter()
    h = jitmod.load_kernel(k.name, k.cubin(), compiled.dev_index)
    compiled.wait_seconds += time.perf_counter() - t0
    compiled.kernels[di] = h
    return h


def _prof_begin():
    if _prof_log is None:
        return None
    ev = torch.cuda.Event(enable_timing=True)
    ev.record()
    return ev


def _prof_end(ev, di: int, nbytes: int) -> None:
    if ev is not None:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        _prof_log.append((di, nbytes, ev, e1))


def _run_descs(compiled, first, count, state, rows_eff, L, norms, grid_limit, stream,
               skip=()) -> int:
    """Launch sweeps first .. first+count-1; returns the number of kernel launches."""
    lib = _native.load()
    if not count:
        return 0
    descs = compiled.descs[first:first + count]
    nptr = norms.data_ptr() if norms is not None else None
    if compiled.kernels is None:
        ev = _prof_begin()
        rc = lib.svb_run_sweeps(state.buf.data_ptr(), rows_eff, L, compiled.blob.data_ptr(),
                                descs.ctypes.data, count, nptr, grid_limit, stream)
        _native.check(rc, "svb_run_sweeps")
        _prof_end(ev, first, sum(compiled.desc_bytes[first:first + count]))
        return count
    launches = 0
    for i in range(count):
        if first + i in skip:
            continue
        cb = compiled.cbits.get(first + i)
        if cb:  # a kernel compiled for part launches: run all parts in order
            for c in range(1 << len(cb)):
                _launch_part(compiled, first + i, state, norms, grid_limit, stream, cb, c)
            launches += 1 << len(cb)
            continue
        ev = _prof_begin()
        rc = lib.svb_jit_launch_sweep(_kernel(compiled, first + i), state.buf.data_ptr(),
                                      compiled.blob.data_ptr(), descs[i:i + 1].ctypes.data, nptr,
                                      grid_limit, stream)
        _native.check(rc, "svb_jit_launch_sweep")
        _prof_end(ev, first + i, compiled.desc_bytes[first + i])
        launches += 1
    return launches


def _alpha(st, geo: prog.DeviceGeometry) -> int:
    """This process's id bits at a remap's swapped rank bits (selector order)."""
    me = geo.rank_base >> geo.h
    alpha = 0
    for ib, _ in st.swaps:
        alpha = (alpha << 1) | ((me >> (ib - geo.h)) & 1)
    return alpha


def _broadcast_merges(dp, geo: prog.DeviceGeometry, sparse: dict, ld_xor: dict, st_keep: dict,
                      overlap: dict) -> dict:
    """Sparse sweeps whose only work is H on dead bits (plus constant
    scales) merged into the sweep before them.

    From |0...0>, a sweep j+1 whose every op is an H on a tile bit that is
    still dead (all amplitudes with that bit set are zero) or a constant
    scale just copies each amplitude v at position P (bits F clear) to the
    2^|F| positions P | f, times the scale c: with x1 = 0 an H butterfly
    (twiddles act on x1 only) gives x0 on both sides.  If its store keeps
    every bit in place and it wakes every dead bit of its tile, sweep j can
    write c * v to those positions directly and sweep j+1 is not launched
    (QFT-30: the last sweep reads 4.3 GB and writes 17.2 GB to expand two
    never-touched qubits).  Returns {j: (F mask, c, norm offset, norm slot
    of j)}: the merged kernel adds sum |v|^2 at its norm slot when j ends a
    leaf and 2^|F| sum |c v|^2 at slot + offset for j+1's leaf."""
    out = {}
    order = []  # launch order; None = a step between sweeps (remap, unfolded localize)
    for st in dp.steps:
        if st.kind in ("sweeps", "materialize"):
            order.extend(range(st.first, st.first + st.count))
        elif not (st.kind == "localize" and st.folded):  # a folded localize moves nothing
            order.append(None)
    chunked = set(overlap) | {i for i, d in enumerate(dp.buf.descs) if d.get("cbits")}
    for j, j1 in zip(order, order[1:]):
        if j is None or j1 is None or j1 != j + 1 or j in out or (j - 1) in out:
            continue
        if j not in sparse or j1 not in sparse or sparse[j][1] or sparse[j][0] is None:
            continue
        if {j, j1} & chunked or j in ld_xor or j1 in st_keep:
            continue
        m = _broadcast_only(dp, j1, sparse[j1], geo.D)
        if m is None:
            continue
        fmask, c = m  # c: combination -> constants
        # across a folded localized remap: sweep j keeps region alpha of the
        # swapped bits and sweep j+1 reads it through a load XOR; when the
        # broadcast covers those bits, storing each kept value at every
        # combination of them (the region bits cleared) is the same
        if j in st_keep and st_keep[j][0] & ~fmask:
            continue
        if j1 in ld_xor and ld_xor[j1] & ~fmask:
            continue
        slot_j, slot_1 = int(dp.buf.descs[j]["norm_slot"]), int(dp.buf.descs[j1]["norm_slot"])
        if slot_j >= 0 and slot_1 >= 0:
            out[j] = (fmask, c, slot_1 - slot_j, slot_j)
        elif slot_1 >= 0:
            out[j] = (fmask, c, 0, slot_1)
        else:
            out[j] = (fmask, c, None, slot_j)
    return out


def _broadcast_only(dp, i: int, sparse_i: tuple, D: int):
    """(F mask, {f: constants}) when sweep i only expands dead bits (see
    _broadcast_merges), else None.

    The op list is replayed on the one nonzero input of each group (x0,
    every dead-bit combination zero): an H (fused or not; twiddles act on
    the zero half) copies x0 to both sides, a 2x2 / 4x4 on dead bits sends
    x0 times its first column to the combinations, an X moves it, a phase
    anchored on a dead bit touches only zeros, and scales multiply every
    copy.  Each combination f keeps the constants in the order the sweep
    would multiply them (the merged store repeats them, so the values are
    bit-identical); a combination missing from the map is zero."""
    supp, full_out = sparse_i
    d = dp.buf.descs[i]
    K = int(d["K"])
    tin = [int(b) for b in d["tin"][:K]]
    sw = [int(x) for x in d["sw"][:K]]
    tout = {sw.index(int(d["st_sw"][q])): int(d["st_dev"][q]) for q in range(K)}
    if int(d["st_flip"]) or d.get("cbits"):
        return None
    tinmask = sum(1 << b for b in tin)
    if supp is None or (full_out and (supp | tinmask) != (1 << D) - 1):
        return None  # it would also write zeros outside its live tiles
    dead = tinmask & ~supp
    ops = dp.buf.ops[d["op_begin"]: d["op_begin"] + d["op_count"]]
    coef = dp.buf.coef
    regs, woke = None, 0
    copies = {0: []}  # combination of woken bits -> constants applied to x0

    def fresh(slot):
        b = tin[regs[slot]]
        return b if (dead >> b) & 1 and not (woke >> b) & 1 else None

    for o in ops:
        kind = int(o["kind"])
        if kind == prog.OP_STAGE:
            rm = int(o["rmask"])
            regs = [k for k in range(K) if (rm >> k) & 1]
            continue
        if int(o["pmask"]) or regs is None:
            return None
        if kind in (prog.OP_H, prog.OP_U1, prog.OP_X):
            b = fresh(int(o["a"]))
            if int(o["rmask"]) or b is None:  # controlled, or on a live bit: real mixing
                return None
            bit = 1 << b
            if kind == prog.OP_H:
                copies = {**copies, **{f | bit: list(ch) for f, ch in copies.items()}}
            elif kind == prog.OP_X:
                copies = {f | bit: ch for f, ch in copies.items()}
            else:
                m00, m10 = complex(coef[int(o["coef"])]), complex(coef[int(o["coef"]) + 2])
                nxt = {}
                for f, ch in copies.items():
                    if m00 != 0:
                        nxt[f] = ch + [m00]
                    if m10 != 0:
                        nxt[f | bit] = ch + [m10]
                copies = nxt
            woke |= bit
        elif kind == prog.OP_U2:
            ba, bb = fresh(int(o["a"])), fresh(int(o["b"]))
            if ba is None or bb is None:
                return None
            M = np.asarray(coef[int(o["coef"]): int(o["coef"]) + 16]).reshape(4, 4)
            nxt = {}
            for f, ch in copies.items():
                for r in range(4):  # rows in _emit_op order: (b, a) = (r & 1, r >> 1)
                    if M[r, 0] != 0:
                        nxt[f | ((r & 1) << bb) | ((r >> 1) << ba)] = ch + [complex(M[r, 0])]
            copies = nxt
            woke |= (1 << ba) | (1 << bb)
        elif kind == prog.OP_PH:
            if fresh(int(o["a"])) is None:  # a phase on amplitudes that can be nonzero
                return None
        elif kind == prog.OP_SCALE:
            cs = complex(coef[int(o["coef"])])
            copies = {f: ch + [cs] for f, ch in copies.items()}
        elif kind == prog.OP_PHALL:
            if int(o["ctab"]) >= 0 or int(o["tab"]) >= 0 or int(o["tf"]) >= 0:
                return None
            cp = complex(coef[int(o["coef"])])
            if cp != 1:
                copies = {f: ch + [cp] for f, ch in copies.items()}
        else:
            return None
    if not woke or woke != dead:
        return None
    # the store may permute the woken bits among themselves (a final relabel);
    # every other bit must stay in place
    for k in range(K):
        if (woke >> tin[k]) & 1:
            if not (woke >> tout[k]) & 1:
                return None
        elif tout[k] != tin[k]:
            return None
    out_bit = {tin[k]: tout[k] for k in range(K)}
    moved = {}
    for f, ch in copies.items():
        moved[sum(1 << out_bit[b] for b in range(D) if (f >> b) & 1)] = ch
    return woke, moved


def _fold_localize(dp, geo: prog.DeviceGeometry, sparse: dict) -> dict:
    """Localized remaps whose next sweep is sparse and holds every swapped
    local bit in its tile: that sweep reads region alpha through an XOR of
    its load addresses (no region move).  Returns {descriptor: xor mask} and
    marks the steps folded."""
    out = {}
    steps = dp.steps
    for i, st in enumerate(steps):
        if st.kind != "localize":
            continue
        nxt = next((x for x in steps[i + 1:] if x.kind in ("sweeps", "materialize") and x.count), None)
        if nxt is None or nxt.first not in sparse:
            continue
        d = dp.buf.descs[nxt.first]
        tin = set(int(b) for b in d["tin"][:d["K"]])
        if not all(lb in tin for _, lb in st.swaps):
            continue
        alpha, m, mask = _alpha(st, geo), len(st.swaps), 0
        for j, (_, lb) in enumerate(st.swaps):
            if (alpha >> (m - 1 - j)) & 1:
                mask |= 1 << lb
        if mask:
            out[nxt.first] = mask
        st.folded = True
    return out


def _prefix_store_masks(dp, geo: prog.DeviceGeometry, sparse: dict) -> dict:
    """The last sweep of a replicated prefix stores only this process's
    region alpha of the swapped local bits when those bits are its tile bits
    (the other regions are never read again): {descriptor: (mask, value)}."""
    out = {}
    steps = dp.steps
    for i, st in enumerate(steps):
        if st.kind != "localize":
            continue
        prev = next((x for x in reversed(steps[:i]) if x.kind in ("sweeps", "materialize") and x.count), None)
        if prev is None:
            continue
        di = prev.first + prev.count - 1
        d = dp.buf.descs[di]
        if di not in sparse or sparse[di][1]:  # full_out sweeps write every position
            continue
        tin = set(int(b) for b in d["tin"][:d["K"]])
        if not all(lb in tin for _, lb in st.swaps):
            continue
        alpha, m = _alpha(st, geo), len(st.swaps)
        mask = val = 0
        for j, (_, lb) in enumerate(st.swaps):
            mask |= 1 << lb
            if (alpha >> (m - 1 - j)) & 1:
                val |= 1 << lb
        out[di] = (mask, val)
    return out


def _localize(state: _State, st, geo: prog.DeviceGeometry, stream) -> int:
    """The remap after a replicated sparse prefix (program.localize_applies):
    this process holds the prefix state of the process with the unit
    amplitude, and after the reference's Pack/Exchange/Unpack it would hold
    that state's region alpha (its own id bits at the swapped rank bits,
    executor.py:235-243) at region 0 of the swapped local bits, zeros
    elsewhere.  Region alpha moves to region 0 in HBM; the other regions are
    left stale and read as zeros by the next (sparse) sweep."""
    lib = _native.load()
    alpha = _alpha(st, geo)
    lbits = [lb for _, lb in st.swaps]
    if alpha == 0 or getattr(st, "folded", False):  # folded: the next sweep reads region alpha
        return 0
    flat = _Flat(state)
    arr, l32 = _native.i32_array(lbits)
    _native.check(lib.svb_region_move(state.buf.data_ptr(), flat.L, l32, len(lbits), alpha, 0, stream),
                  "svb_region_move")
    return 1


def _remap(state: _State, swaps: list, geo: prog.DeviceGeometry, group, stream) -> int:
    """Pairwise bit swaps rank bit <-> physical local bit (executor.py:224-281).

    `swaps` are (rank integer bit, physical local device bit) from the schedule.
    """
    lib = _native.load()
    L, g, h = geo.L, geo.g, geo.h
    local_u, local_w, remote = [], [], []
    for ib, lb in swaps:
        if ib < h:
            local_u.append(L + ib)
            local_w.append(lb)
        else:
            remote.append((ib - h, lb))
    launches = 0
    if local_u:
        D = L + h
        if (state.rows << L) < prog.NREG:
            D = max(D, 4)
        u_arr = np.asarray(local_u, dtype=np.int32)
        w_arr = np.asarray(local_w, dtype=np.int32)
        _native.check(
            lib.svb_bitswap(state.buf.data_ptr(), D, u_arr.ctypes.data_as(_native._pi32),
                            w_arr.ctypes.data_as(_native._pi32), len(local_u), stream),
            "svb_bitswap",
        )
        launches += 1
    if remote:
        from . import comm

        flat = _Flat(state)
        if state.ctx is not None:
            launches += comm.peer_exchange(flat, remote, state.ctx, stream, state.ctx.next_epoch())
        else:
            launches += comm.exchange(flat, remote, geo, group)
    return launches


# ---------------------------------------------------------------------------
# layout / verification helpers
# ---------------------------------------------------------------------------


def _all_blocks(state: DistState) -> torch.Tensor:
    if state.world == 1:
        return state.blocks
    import torch.distributed as dist

    parts = [torch.empty_like(state.blocks) for _ in range(state.world)]
    dist.all_gather(parts, state.blocks.contiguous(), group=state.group)
    return torch.cat(parts, dim=0)


@_on_device(lambda state, *a, **k: _arg_device(state))
def gather_device(state: DistState) -> torch.Tensor:
    """Dense qubit-0-most-significant vector on the device (executor.py:320-326)."""
    blocks = _all_blocks(state)
    layout = state.layouts[state.phase]
    d = state.d
    dense = torch.empty(1 << d, dtype=torch.complex128, device=blocks.device)
    if d == 0:
        dense.copy_(blocks.reshape(-1))
        return dense
    _bitperm(blocks.contiguous().view(-1), dense, _storage_bitperm(layout, d, to_basis=True))
    return dense


GATHER_CHUNK_BITS = int(os.environ.get("SVB200_GATHER_CHUNK_BITS", "22"))  # 64 MiB chunks


def gather(state: DistState, root: int | None = None) -> np.ndarray | None:
    """Dense host vector, like the reference's gather (executor.py:320-326).

    A sharded state is assembled chunk by chunk in host memory: every
    process reads its shard in basis-sorted order one 2^22-amplitude chunk
    at a time (svb_gather_bits), the chunks are all-gathered (gathered to
    `root` when given) and written into the dense vector through a strided
    view, so no GPU ever holds more than its shard plus world chunks.  With
    root, processes other than root return None.  One large single-GPU
    state takes the same chunked path (no second full-size device buffer)."""
    big = (16 << state.d) > (1 << 33)  # > 8 GiB: avoid a full-size device copy
    if state.world == 1 and not big:
        return gather_device(state).cpu().numpy()
    return _gather_chunked(state, root)


@_on_device(lambda state, *a, **k: _arg_device(state))
def _gather_chunked(state: DistState, root: int | None) -> np.ndarray | None:
    import torch.distributed as dist

    from . import sampling

    lib = _native.load()
    d, g, world = state.d, state.g, state.world
    blocks = state.blocks.contiguous()
    rows = blocks.shape[0]
    layout = state.layouts[state.phase]
    me = state.rank_base // rows
    want = root is None or root == me
    dense = np.empty(1 << d, dtype=np.complex128) if want else None
    view = dense.reshape((2,) * d) if want and d else dense
    geos = [sampling.shard_geometry(layout, d, g, rows, p * rows) for p in range(world)]
    D, perm, _, _ = geos[me]
    inv = [0] * D  # sorted bit -> storage bit
    for s_, j in enumerate(perm):
        inv[j] = s_
    arr, inv32 = _native.i32_array(inv)
    c = min(D, GATHER_CHUNK_BITS)
    stage = torch.empty(1 << c, dtype=torch.complex128, device=blocks.device)
    bufs = [torch.empty_like(stage) for _ in range(world)] if world > 1 else [stage]
    stream = _stream_ptr(blocks.device)

    def place(p, k, host):
        Dp, _, fm, fv = geos[p]
        idx = []
        for axis in range(d):  # axis 0 = basis bit d-1 (qubit 0)
            bit = d - 1 - axis
            idx.append(((fv >> bit) & 1) if (fm >> bit) & 1 else slice(None))
        sub = view[tuple(idx)] if d else view
        lead = tuple((k >> (Dp - c - 1 - i)) & 1 for i in range(Dp - c))
        sub[lead] = host.reshape((2,) * c) if c else host

    for k in range(1 << (D - c)):
        _native.check(lib.svb_gather_bits(blocks.data_ptr(), D, inv32, k << c, 1 << c, stage.data_ptr(), stream),
                      "svb_gather_bits")
        if world > 1:
            if root is None or dist.get_backend(state.group) == "gloo":
                dist.all_gather(bufs, stage, group=state.group)
            else:
                dist.gather(stage, bufs if want else None, dst=root, group=state.group)
        if want:
            for p in range(world):
                place(p, k, bufs[p].cpu().numpy())
    return dense


@_on_device(lambda dense, plan, phase=0, device=None, **k: device or _arg_device(dense))
def scatter(dense, plan, phase: int = 0, device=None, local_perm=None) -> DistState:
    """Distribute a dense state into rank blocks at the given layout phase (executor.py:329-343).

    `local_perm` (internal) additionally places reference local bit r at
    physical bit local_perm[r] (the executor's initial layout).
    """
    device = _require_cuda(device)
    d, g = plan.d, plan.g
    shape = tuple(dense.shape)
    if shape != (1 << d,):
        raise DimensionMismatch(f"state length {shape} != 2^{d}")
    if isinstance(dense, torch.Tensor):
        src = dense.to(device=device, dtype=torch.complex128).contiguous()
    else:
        src = torch.from_numpy(np.ascontiguousarray(dense, dtype=np.complex128)).to(device)
    layout = plan.layout_phases[phase]
    flat = torch.empty(1 << d, dtype=torch.complex128, device=device)
    if d == 0:
        flat.copy_(src)
    else:
        perm = _storage_bitperm(layout, d, to_basis=False)
        if local_perm is not None:
            L = d - g
            perm = [local_perm[p] if p < L else p for p in perm]
        _bitperm(src, flat, perm)
    return DistState(
        blocks=flat.view(1 << g, 1 << (d - g)), phase=phase, d=d, g=g,
        layouts=[list(p) for p in plan.layout_phases],
    )


def _as_device_vec(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.complex128).contiguous().view(-1)
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128).reshape(-1)).to(device)


def _same_sharding(a, b) -> bool:
    return (isinstance(a, DistState) and isinstance(b, DistState) and a.world > 1 and
            (a.d, a.g, a.world, a.rank_base) == (b.d, b.g, b.world, b.rank_base) and
            list(a.layouts[a.phase]) == list(b.layouts[b.phase]))


def _compare_sharded(a: DistState, b: DistState) -> float:
    """compare() of two states sharded the same way, without gathering: the
    phase is taken at the global argmax of |a||b| (ties to the smallest basis
    index, like numpy's argmax), then the max deviation is all-reduced."""
    import torch.distributed as dist

    lib = _native.load()
    A, B = a.blocks.contiguous().view(-1), b.blocks.contiguous().view(-1)
    device = A.device
    n = A.numel()
    d = a.d
    L = d - a.g
    layout = a.layouts[a.phase]
    perm = [0] * d
    for q in range(d):  # storage bit (LSB-indexed) -> basis bit
        perm[d - 1 - layout[q]] = d - 1 - q
    arr, p32 = _native.i32_array(perm)
    scratch = torch.empty(int(lib.svb_shard_scratch_bytes(n)), dtype=torch.uint8, device=device)
    out = torch.zeros(4, dtype=torch.float64, device=device)
    st = _stream_ptr(device)
    _native.check(lib.svb_shard_argmax(A.data_ptr(), B.data_ptr(), n, a.rank_base << L, d, p32, out.data_ptr(),
                                       scratch.data_ptr(), st), "svb_shard_argmax")
    parts = [torch.empty_like(out) for _ in range(a.world)]
    dist.all_gather(parts, out, group=a.group)
    best = None
    for t in parts:
        w = float(t[0].item())
        bi = int(t[1:2].view(torch.int64).item())
        if best is None or w > best[0] or (w == best[0] and bi < best[1]) or (w != w and best[0] == best[0]):
            best = (w, bi, complex(float(t[2].item()), float(t[3].item())))
    w, _, z = best
    if w != w:  # a NaN amplitude: numpy's argmax picks it and the result is NaN
        return float("nan")
    phi = z / abs(z) if w > 0.0 else 1.0 + 0.0j
    dev = torch.zeros(1, dtype=torch.float64, device=device)
    _native.check(lib.svb_shard_maxdev(A.data_ptr(), B.data_ptr(), n, phi.real, phi.imag, dev.data_ptr(),
                                       scratch.data_ptr(), st), "svb_shard_maxdev")
    dist.all_reduce(dev, op=dist.ReduceOp.MAX, group=a.group)
    return float(dev.item())


@_on_device(lambda a, b, device=None: device or _arg_device(a) or _arg_device(b))
def compare(a, b, device=None) -> float:
    """Max amplitude deviation after aligning global phase at the largest amplitude.

    Dense vectors as in the reference; two DistStates sharded the same way
    over several processes are compared shard by shard (no gather)."""
    if _same_sharding(a, b):
        return _compare_sharded(a, b)
    if isinstance(a, DistState):
        a = gather_device(a)
    if isinstance(b, DistState):
        b = gather_device(b)
    if tuple(a.shape) != tuple(b.shape):
        raise DimensionMismatch(f"{tuple(a.shape)} vs {tuple(b.shape)}")
    device = _require_cuda(device if device is not None else (a.device if isinstance(a, torch.Tensor) and a.is_cuda else None))
    lib = _native.load()
    A, B = _as_device_vec(a, device), _as_device_vec(b, device)
    n = A.numel()
    scratch = torch.empty(int(lib.svb_compare_scratch_bytes(n)), dtype=torch.uint8, device=device)
    out = torch.zeros(1, dtype=torch.float64, device=device)
    _native.check(lib.svb_compare(A.data_ptr(), B.data_ptr(), n, out.data_ptr(), scratch.data_ptr(),
                                  _stream_ptr(device)), "svb_compare")
    return float(out.item())


@_on_device(lambda a, b, device=None: device or _arg_device(a) or _arg_device(b))
def fidelity(a, b, device=None) -> float:
    """|<a|b>|^2 / (<a|a><b|b>) on the device (sharded DistStates: per shard, then all-reduced)."""
    if _same_sharding(a, b):
        import torch.distributed as dist

        A, B = a.blocks.reshape(-1), b.blocks.reshape(-1)
        ov = torch.vdot(A, B)
        t = torch.stack([ov.real, ov.imag, torch.vdot(A, A).real, torch.vdot(B, B).real])
        dist.all_reduce(t, group=a.group)
        re, im, na, nb = (float(x) for x in t.tolist())
        return (re * re + im * im) / (na * nb)
    if isinstance(a, DistState):
        a = gather_device(a)
    if isinstance(b, DistState):
        b = gather_device(b)
    device = _require_cuda(device)
    A, B = _as_device_vec(a, device), _as_device_vec(b, device)
    ov = torch.vdot(A, B)
    return float((ov.abs() ** 2 / (torch.vdot(A, A).real * torch.vdot(B, B).real)).item())


@_on_device(lambda dense, shots, seed, device=None: device or _arg_device(dense))
def sample(dense, shots: int, seed: int | None, device=None) -> dict:
    """Seeded measurement histogram {bitstring: count}, qubit 0 first
    (executor.py:375-383), computed on the GPU by ``sampling.sample_state``:
    the same numpy Generator uniforms and CDF inversion over the basis order.

    `dense` is a dense vector (host or device) or a DistState (sharded ones
    are sampled in place, collectively)."""
    from . import sampling

    if isinstance(dense, DistState):
        return sampling.sample_state(dense, shots, seed)
    device = _require_cuda(device if device is not None else
                           (dense.device if isinstance(dense, torch.Tensor) and dense.is_cuda else None))
    vec = _as_device_vec(dense, device)
    n = vec.numel()
    d = n.bit_length() - 1
    if n != 1 << d:
        raise DimensionMismatch(f"state length {n} is not a power of two")
    st = DistState(blocks=vec.view(1, n), phase=0, d=d, g=0, layouts=[list(range(d))])
    return sampling.sample_state(st, shots, seed)


@_on_device(lambda circuit, device=None: device)
def oracle_simulate(circuit, device=None) -> np.ndarray:
    """Dense reference-order simulation from |0...0>, on the GPU (executor.py:346-358)."""
    from . import kernels

    d = circuit.num_qubits
    if d > 14:
        raise TooLarge(f"oracle capped at 14 qubits, got {d}")
    device = _require_cuda(device)
    state = torch.zeros((1, 1 << d), dtype=torch.complex128, device=device)
    state[0, 0] = 1.0
    for op in circuit.ops:
        mat = np.asarray(op.gate.matrix)
        kernels.apply_gate(state, mat, list(op.qubits))
    return state.view(-1).cpu().numpy()
