"""Host compiler: ApplyFused payload -> device sweep program (ops + tables).

This replaces the reference's per-gate interpretation of an ApplyFused leaf
(``svpart/executor.py:123-176``) with a one-time translation into the
program format consumed by the fused sweep kernel (``csrc/sweep.cu``, ABI in
``include/svb200.h``).  The semantics it must reproduce, gate by gate:

* positions: ``pos = layout[q]``; ``pos < g`` is a rank ("global") slot,
  otherwise local bit ``pos - g`` with stride ``2^(L-1-(pos-g))``
  (``plan.py:3-8``); a stale passthrough mark raises ``PlanInvalid``
  (``executor.py:129-131``);
* a diagonal gate with global slots applies, per rank, the sub-diagonal with
  those slots fixed to the rank's bits (``executor.py:142-157``);
* a non-diagonal gate with global slots must have them all as controls
  (``executor.py:159-162``) and then acts, on ranks whose global controls are
  all 1, as the matrix restricted to control=1 (``executor.py:163-176``).

Device coordinates: a device holds ``rows = 2^h`` consecutive ranks as rows
of one array, so its amplitudes are addressed by a D = L + h bit "device
index" ``row * 2^L + local`` (bits counted from the LSB).  Rank bits below h
are row bits (device bits L..D-1); higher rank bits are constant on the
device and are resolved here, so each device gets its own program.

Within a sweep a 2^K-amplitude tile (K tile bits) is processed per CTA; all
other device bits are "fixed" bits F.  Dense gates need their targets in the
tile; diagonal gates are decomposed into phase factors [bits all 1] -> c and
commuted forward until a dense gate touches one of their bits ("flush"), where
they are fused into that gate's pre-phase.  SWAP and uncontrolled X are
virtual (relabel / flip the tile bit and fix it up in the store mapping).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import os

import numpy as np

from . import gates as gatelib
from .errors import PlanInvalid

KMAX = 12  # tile bits per sweep (2 x 64 KB double-buffered in shared memory)
RB = 4  # register slots per thread
NREG = 1 << RB

OP_STAGE, OP_U1, OP_H, OP_X, OP_U2, OP_PH, OP_PHALL, OP_SCALE = 1, 2, 3, 4, 5, 6, 7, 8
F_PHASE = 1
F_PREG_SHIFT = 4
F_TORDER = 1 << 8  # OP_STAGE: pval holds the stage's thread-bit order (4 bits per thread bit)

OP_DTYPE = np.dtype(
    [
        ("kind", "<i4"), ("a", "<i4"), ("b", "<i4"), ("rmask", "<u4"),
        ("pmask", "<u8"), ("pval", "<u8"),
        ("coef", "<i4"), ("tab", "<i4"), ("ctab", "<i4"), ("tf", "<i4"),
        ("flags", "<i4"), ("pad", "<i4", (3,)),
    ]
)
CTERM_DTYPE = np.dtype([("dst", "<i4"), ("pad", "<i4"), ("mask", "<u8"), ("re", "<f8"), ("im", "<f8")])
MAXT = 13
DESC_DTYPE = np.dtype(
    [
        ("K", "<i4"), ("D", "<i4"),
        ("tin", "<i4", (MAXT,)), ("sw", "<i4", (MAXT,)),
        ("st_dev", "<i4", (MAXT,)), ("st_sw", "<i4", (MAXT,)),
        ("st_flip", "<u8"),
        ("op_begin", "<i4"), ("op_count", "<i4"),
        ("nctab", "<i4"), ("norm_slot", "<i4"),
        ("rb", "<i4"), ("groups", "<i4"),
        ("ops_off", "<i8"), ("coef_off", "<i8"), ("tab_off", "<i8"),
        ("cterm_off", "<i8"), ("cofs_off", "<i8"),
    ],
    align=True,
)
assert OP_DTYPE.itemsize == 64 and CTERM_DTYPE.itemsize == 32

_H = np.array([[1, 1], [1, -1]], dtype=np.complex128) / math.sqrt(2)
_X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
_I2 = np.eye(2, dtype=np.complex128)


@dataclass
class DeviceGeometry:
    """Which slice of the distributed state one device holds."""

    d: int
    g: int
    h: int  # log2(rows on this device)
    rank_base: int  # global rank id of row 0 (multiple of 2^h)
    pad_to: int = 0  # tiny states are padded with phantom bits to this many

    @property
    def L(self) -> int:
        return self.d - self.g

    @property
    def D(self) -> int:
        return max(self.L + self.h, self.pad_to)


# ---------------------------------------------------------------------------
# 1. gate resolution: payload entry -> primitive ops in device-bit terms
# ---------------------------------------------------------------------------


@dataclass
class Dense1:
    """2x2 on device bit `bit`, applied where all `ctrl` bits equal their value."""

    bit: int
    m: np.ndarray
    ctrl: dict  # device bit -> required value (0/1)
    noop: bool = False  # a constant-0 control made it identity on this device
    perm: bool = False  # structurally a bit flip (x, cx, ccx): costs no FP64
    gctl: bool = False  # had rank-global controls (resolved differently per device)


@dataclass
class Dense2:
    """4x4 on device bits (a, b); matrix index bit 1 <-> a, bit 0 <-> b."""

    a: int
    b: int
    m: np.ndarray


@dataclass
class Swap:
    a: int
    b: int


@dataclass
class ExchMark:
    """Marker in the planning stream: these reference local bits are exchanged next."""

    bits: tuple


@dataclass
class Factor:
    """Diagonal factor: multiply by c where every bit in `bits` is 1 (0-2 bits)."""

    bits: tuple
    c: complex


def _slot_device_bit(pos: int, geo: DeviceGeometry):
    """(device_bit, None) for a bit that varies on this device, or (None, value)."""
    if pos >= geo.g:
        return geo.L - 1 - (pos - geo.g), None
    ib = geo.g - 1 - pos  # integer bit of the rank id
    if ib < geo.h:
        return geo.L + ib, None
    return None, (geo.rank_base >> ib) & 1


def _decompose_diag(diag: np.ndarray, bits: list) -> list:
    """Exact multiplicative decomposition of a <=2-bit diagonal into Factors."""
    p = len(bits)
    if p == 0:
        return [Factor((), complex(diag[0]))]
    if p == 1:
        d0, d1 = complex(diag[0]), complex(diag[1])
        out = [Factor((), d0)] if d0 != 1 else []
        r = d1 / d0 if d0 != 1 else d1
        if r != 1:
            out.append(Factor((bits[0],), r))
        return out
    if p == 2:
        # slot 0 = matrix bit 1 (MSB), slot 1 = matrix bit 0
        d00, d01, d10, d11 = (complex(x) for x in diag)
        out = []
        if d00 != 1:
            out.append(Factor((), d00))
        c0 = d10 / d00 if d00 != 1 else d10  # slot0 alone
        c1 = d01 / d00 if d00 != 1 else d01  # slot1 alone
        if c0 != 1:
            out.append(Factor((bits[0],), c0))
        if c1 != 1:
            out.append(Factor((bits[1],), c1))
        num = d11 * d00 if d00 != 1 else d11
        den = d10 * d01
        c01 = num / den if den != 1 else num
        if c01 != 1:
            out.append(Factor((bits[0], bits[1]), c01))
        return out
    raise NotImplementedError("diagonal gates wider than 2 device bits are not supported")


def _controlled_split(m: np.ndarray, ctl_slots: list, p: int):
    """If m acts as identity unless all control slots are 1, return the target block."""
    if not ctl_slots:
        return None
    dim = 1 << p
    ones = 0
    for s in ctl_slots:
        ones |= 1 << (p - 1 - s)
    inside = [i for i in range(dim) if (i & ones) == ones]
    outside = [i for i in range(dim) if (i & ones) != ones]
    for i in outside:
        row = m[i]
        if row[i] != 1 or np.count_nonzero(row) != 1:
            return None
        if np.count_nonzero(m[:, i]) != 1:
            return None
    return m[np.ix_(inside, inside)]


def resolve_entry(entry: dict, layout, geo: DeviceGeometry) -> list:
    """Primitive ops for one payload gate, in device-bit terms (executor.py:125-176)."""
    gate = gatelib.gate(entry["kind"], tuple(entry["params"]))
    qubits = list(entry["qubits"])
    positions = [layout[q] for q in qubits]
    global_slots = [i for i, pos in enumerate(positions) if pos < geo.g]
    if bool(global_slots) != bool(entry["passthrough"]):
        raise PlanInvalid(f"stale passthrough mark on {entry}")
    p = gate.num_qubits
    if not gate.is_diagonal and global_slots and not set(global_slots) <= gate.controls:
        raise PlanInvalid(f"{gate.kind} on {qubits} has a non-control global slot")

    slot_bit, slot_const = [], []
    for pos in positions:
        b, c = _slot_device_bit(pos, geo)
        slot_bit.append(b)
        slot_const.append(c)
    fixed = [i for i in range(p) if slot_bit[i] is None]
    free = [i for i in range(p) if slot_bit[i] is not None]

    if gate.is_diagonal:
        diag = np.asarray(gate.matrix).diagonal().reshape((2,) * p) if p else np.asarray(gate.matrix).diagonal()
        idx = tuple(slot_const[i] if i in fixed else slice(None) for i in range(p))
        sub = np.asarray(diag[idx]).reshape(-1)
        return _decompose_diag(sub, [slot_bit[i] for i in free])

    # non-diagonal: fixed slots are controls (validated above); a constant-0
    # control makes the gate the identity on this device, but it is kept as a
    # placeholder with the same structure so every device plans the same
    # tiles, fusions and layouts
    noop = any(slot_const[i] == 0 for i in fixed)
    m = np.asarray(gate.matrix).reshape((2,) * (2 * p))
    idx = [slice(None)] * (2 * p)
    for i in fixed:
        idx[i] = 1
        idx[p + i] = 1
    k = len(free)
    sub = np.ascontiguousarray(m[tuple(idx)].reshape(1 << k, 1 << k))
    free_bits = [slot_bit[i] for i in free]
    ctl = [j for j, i in enumerate(free) if i in gate.controls]
    tgt = [j for j in range(k) if j not in ctl]
    if k == 2 and not ctl and gate.kind == "swap":
        if noop:
            raise PlanInvalid(f"swap on {qubits} has a global slot")
        return [Swap(free_bits[0], free_bits[1])]
    block = _controlled_split(sub, ctl, k) if ctl else None
    if block is not None and len(tgt) == 1:
        perm = bool(np.array_equal(block, _X))
        return [Dense1(free_bits[tgt[0]], np.eye(2, dtype=np.complex128) if noop else block,
                       {} if noop else {free_bits[j]: 1 for j in ctl}, noop=noop, perm=perm,
                       gctl=bool(fixed))]
    if k == 1:
        perm = bool(np.array_equal(sub, _X))
        return [Dense1(free_bits[0], np.eye(2, dtype=np.complex128) if noop else sub, {},
                       noop=noop, perm=perm, gctl=bool(fixed))]
    raise NotImplementedError(f"no device decomposition for {gate.kind} on {k} free slots")


# ---------------------------------------------------------------------------
# 2. sweep assembly
# ---------------------------------------------------------------------------


@dataclass
class _Item:
    """A register-level operation before stage assignment (physical tile bits)."""

    kind: int
    bits: tuple  # physical tile-local positions needing register slots
    m: np.ndarray | None = None
    ctrl: dict = field(default_factory=dict)  # physical device bit -> value
    factors: list = field(default_factory=list)  # pre-phase factors (physical device bits)
    h_scaled: bool = False


@dataclass
class SweepProgram:
    K: int
    tin: list  # tile-local k -> physical device bit (sorted)
    items: list
    out_map: dict  # physical tile bit -> (destination device bit, flip)
    norm_slot: int = -1
    scale: complex = 1.0


LOW_RUN_BITS = 4  # every tile spans physical bits 0..3: 256 B contiguous runs


def _needs(prim) -> list:
    """Reference bits a primitive needs inside the tile (dense targets, virtual flips)."""
    if isinstance(prim, Dense1):
        return [prim.bit]
    if isinstance(prim, Dense2):
        return [prim.a, prim.b]
    return []


# ---------------------------------------------------------------------------
# 1b. gate fusion (structural, identical on every device)
# ---------------------------------------------------------------------------


def _embed2(pr, a: int, b: int) -> np.ndarray:
    """4x4 of a Dense1 / Factor acting inside the bit pair (a = index bit 1)."""
    pos = {a: 1, b: 0}
    out = np.zeros((4, 4), dtype=np.complex128)
    if isinstance(pr, Factor):
        d = np.ones(4, dtype=np.complex128)
        for i in range(4):
            if all((i >> pos[x]) & 1 for x in pr.bits):
                d[i] = pr.c
        return np.diag(d)
    if pr.noop:
        return np.eye(4, dtype=np.complex128)
    tb = pos[pr.bit]
    for i in range(4):
        if not all(((i >> pos[c]) & 1) == v for c, v in pr.ctrl.items()):
            out[i, i] = 1
            continue
        ti = (i >> tb) & 1
        for tj in range(2):
            j = (i & ~(1 << tb)) | (tj << tb)
            out[i, j] = pr.m[ti, tj]
    return out


def _bits_of(pr) -> set:
    if isinstance(pr, Dense1):
        return {pr.bit} | set(pr.ctrl)
    if isinstance(pr, Dense2):
        return {pr.a, pr.b}
    if isinstance(pr, Factor):
        return set(pr.bits)
    if isinstance(pr, Swap):
        return {pr.a, pr.b}
    return set()


# the last sweep before a remap reserves tile room to park the remap's qubits on top
PARK_FIRST = os.environ.get("SVB200_PARK_FIRST", "1") not in ("0", "false", "no")
# pair blocks of bit flips and phases whose flips cancel become phases (fuse_prims)
DIAG_PAIRS = os.environ.get("SVB200_DIAG_PAIRS", "1") not in ("0", "false", "no")


def fuse_prims(prims: list, owners: list | None = None):
    """Merge runs of gates confined to one qubit pair into a single 4x4 (e.g.
    the u,u,cx,u,u,cx,u,u,cx,u,u form of an SU(4)).

    Blocks on disjoint pairs stay open concurrently (gates on disjoint bits
    commute).  A block is fused when it holds at least two non-permutation
    dense gates; otherwise its gates are emitted unchanged (phases and bit
    flips are cheaper than a 4x4).  The decision depends only on gate
    structure, never on device-specific constants.

    A fused block takes the place of its last gate: primitives between its
    gates touch other bits (one touching its pair would have closed it) and
    commute with it, so later sweeps see the gates near their original
    position.

    owners (optional): a tag per primitive (non-decreasing); then returns
    (prims, tags) where a fused primitive carries the tag of its last gate.
    """
    placed: list = []  # (input position, primitive, tag)
    blocks: list = []  # open blocks: dict(bits=set, prims=list, own=list, pos=list)
    tagged = owners is not None
    owners = owners if tagged else [0] * len(prims)

    def close(blk):
        blocks.remove(blk)
        ps = blk["prims"]
        top = blk["own"][-1]
        at = blk["pos"][-1]

        def emit(pr, o, k=None):
            placed.append((at if k is None else k, pr, o))
        dense = [p for p in ps if isinstance(p, Dense1)]
        nonperm = [p for p in dense if not p.perm]
        bits = sorted(blk["bits"])
        if DIAG_PAIRS and len(bits) == 2 and dense and not nonperm and not any(p.gctl for p in dense):
            # bit flips and phases only (QAOA's cx rz cx): when the flips
            # cancel, the block is a diagonal -- phases, no data movement
            # (a runtime-controlled flip is a conditional register swap)
            a, b = bits[1], bits[0]
            m = np.eye(4, dtype=np.complex128)
            for p in ps:
                m = _embed2(p, a, b) @ m
            if not np.any(m - np.diag(np.diag(m))):
                d = np.diag(m)
                for fb, c in (((), d[0]), ((b,), d[1] / d[0]), ((a,), d[2] / d[0]),
                              ((a, b), d[3] * d[0] / (d[1] * d[2]))):
                    if c != 1:
                        emit(Factor(fb, complex(c)), top)
                return
        if len(nonperm) >= 2 and len(bits) == 2:
            a, b = bits[1], bits[0]
            m = np.eye(4, dtype=np.complex128)
            for p in ps:
                m = _embed2(p, a, b) @ m
            emit(Dense2(a, b, m), top)
        elif len(nonperm) >= 2 and len(bits) == 1 and all(not p.ctrl for p in dense):
            (x,) = bits
            m = np.eye(2, dtype=np.complex128)
            for p in ps:
                if isinstance(p, Factor):
                    g = np.diag([1, p.c]) if p.bits else np.eye(2) * p.c
                else:
                    g = np.eye(2, dtype=np.complex128) if p.noop else p.m
                m = g @ m
            emit(Dense1(x, m, {}), top)
        else:
            for p, o, k in zip(ps, blk["own"], blk["pos"]):
                emit(p, o, k)

    for k, (pr, o) in enumerate(zip(prims, owners)):
        bits = _bits_of(pr)
        fusable = isinstance(pr, (Dense1, Factor)) and len(bits) <= 2 and bits
        hit = [blk for blk in blocks if blk["bits"] & bits]
        if fusable and len(hit) > 1 and len(set().union(bits, *(b["bits"] for b in hit))) <= 2:
            # single-qubit blocks on the two bits of this gate (e.g. the u, u
            # before the first cx of an SU(4)) commute and join one block
            items = sorted((kk, pp, oo) for b in hit for kk, pp, oo in zip(b["pos"], b["prims"], b["own"]))
            for b in hit[1:]:
                blocks.remove(b)
            hit = hit[:1]
            hit[0]["bits"] = set().union(*(b["bits"] for b in hit), *(_bits_of(pp) for _, pp, _ in items))
            hit[0]["pos"] = [kk for kk, _, _ in items]
            hit[0]["prims"] = [pp for _, pp, _ in items]
            hit[0]["own"] = [oo for _, _, oo in items]
        if fusable and len(hit) == 1 and len(hit[0]["bits"] | bits) <= 2:
            hit[0]["bits"] |= bits
            hit[0]["prims"].append(pr)
            hit[0]["own"].append(o)
            hit[0]["pos"].append(k)
            continue
        for blk in hit:
            close(blk)
        if fusable and (isinstance(pr, Dense1) or len(bits) == 2):
            blocks.append({"bits": set(bits), "prims": [pr], "own": [o], "pos": [k]})
        else:
            placed.append((k, pr, o))
    for blk in list(blocks):
        close(blk)
    placed.sort(key=lambda x: x[0])
    out = [pr for _, pr, _ in placed]
    return (out, [o for _, _, o in placed]) if tagged else out


def build_sweep(prims: list, tile: list, where: list) -> SweepProgram:
    """Phase scheduling for one sweep.

    `where` maps reference device bit -> physical device bit for the whole
    run and is updated in place by SWAP primitives (a relabeling: no data
    moves).  Uncontrolled X flips a physical tile bit (undone at the store).
    Dense gates act on physical tile bits; diagonal factors are expressed on
    physical bits when they are created and flushed into the next dense gate
    on one of their bits (or into the end-of-sweep phase).
    """
    K = len(tile)
    tile_pos = {b: k for k, b in enumerate(tile)}
    pflip = {b: 0 for b in tile}  # physical tile bit -> value inverted
    pending: list = []  # Factor in physical device bits
    items: list = []
    const = complex(1.0)
    scale = 1.0

    def phys_factor(f: Factor):
        """Reference-bit factor -> physical factors; a flipped bit reads b = 1 - p."""
        nonlocal const
        c = f.c
        bits_p = [where[b] for b in f.bits]
        fl = [pflip.get(pb, 0) for pb in bits_p]
        if not bits_p:
            const *= c
            return []
        if len(bits_p) == 1:
            if fl[0]:  # c^(1-p) = c * (1/c)^p
                const *= c
                return [Factor((bits_p[0],), 1 / c)]
            return [Factor((bits_p[0],), c)]
        a, b = bits_p
        fa, fb = fl
        if not fa and not fb:
            return [Factor((a, b), c)]
        if fa and not fb:  # c^((1-pa) pb) = c^pb * (1/c)^(pa pb)
            return [Factor((b,), c), Factor((a, b), 1 / c)]
        if fb and not fa:
            return [Factor((a,), c), Factor((a, b), 1 / c)]
        # c^((1-pa)(1-pb)) = c * (1/c)^pa * (1/c)^pb * c^(pa pb)
        const *= c
        return [Factor((a,), 1 / c), Factor((b,), 1 / c), Factor((a, b), c)]

    def flush(pb: int) -> list:
        nonlocal pending
        hit = [f for f in pending if pb in f.bits]
        pending = [f for f in pending if pb not in f.bits]
        return hit

    for pr in prims:
        if isinstance(pr, Factor):
            for f in phys_factor(pr):
                if f.bits:
                    pending.append(f)
                else:
                    const *= f.c
            continue
        if isinstance(pr, Swap):
            where[pr.a], where[pr.b] = where[pr.b], where[pr.a]
            continue
        if isinstance(pr, Dense2):
            pa, pb2 = where[pr.a], where[pr.b]
            m = pr.m
            fa, fb = pflip[pa], pflip[pb2]
            if fa or fb:  # conjugate by the pending bit flips
                xa = _X if fa else _I2
                xb = _X if fb else _I2
                f4 = np.kron(xa, xb)
                m = f4 @ m @ f4
            fl = flush(pa) + flush(pb2)
            inside = [f for f in fl if set(f.bits) <= {pa, pb2}]
            for f in fl:
                if f not in inside:
                    anchor = pa if pa in f.bits else pb2
                    items.append(_Item(OP_PH, (tile_pos[anchor],), factors=[f]))
            for f in inside:  # phases on the pair are absorbed into the 4x4
                d = np.ones(4, dtype=np.complex128)
                for i in range(4):
                    bitv = {pa: (i >> 1) & 1, pb2: i & 1}
                    if all(bitv[x] for x in f.bits):
                        d[i] = f.c
                m = m @ np.diag(d)
            items.append(_Item(OP_U2, (tile_pos[pa], tile_pos[pb2]), m=np.array(m)))
            continue
        assert isinstance(pr, Dense1)
        if pr.noop:
            continue
        pb = where[pr.bit]
        m = pr.m
        if pflip[pb]:
            m = _X @ m @ _X
        ctrl = {}
        for cb, val in pr.ctrl.items():
            pc = where[cb]
            ctrl[pc] = val ^ pflip.get(pc, 0)
        if not ctrl and np.array_equal(m, _X):
            pflip[pb] ^= 1  # virtual: relabel the bit value
            continue
        fl = flush(pb)
        if np.array_equal(m, _X):
            if fl:  # the flush must precede the data movement
                items.append(_Item(OP_PH, (tile_pos[pb],), factors=fl))
            items.append(_Item(OP_X, (tile_pos[pb],), ctrl=ctrl))
            continue
        is_h = not ctrl and np.array_equal(m, _H)
        if ctrl and fl:  # a predicated gate cannot carry the (unconditional) pre-phase
            items.append(_Item(OP_PH, (tile_pos[pb],), factors=fl))
            fl = []
        if is_h:
            scale *= 1 / math.sqrt(2)
            items.append(_Item(OP_H, (tile_pos[pb],), factors=fl, h_scaled=True))
        else:
            items.append(_Item(OP_U1, (tile_pos[pb],), m=np.array(m), ctrl=ctrl, factors=fl))

    # leftover phases are applied at the end of the sweep
    items.append(_Item(OP_PHALL, (), factors=pending))
    sp = SweepProgram(K=K, tin=list(tile), items=items,
                      out_map={b: (b, pflip[b]) for b in tile})
    sp.scale = const * scale
    return sp


# ---------------------------------------------------------------------------
# 2b. layout planner: sweep boundaries, tiles and store permutations
# ---------------------------------------------------------------------------


@dataclass
class Step:
    """One step of a device schedule, in plan order."""

    kind: str  # "sweeps" (an ApplyFused task) | "exchange" | "materialize"
    task_id: int | None = None
    first: int = 0  # first descriptor
    count: int = 0  # descriptors
    swaps: list = field(default_factory=list)  # exchange: (rank int bit, physical local bit)
    # exchange overlap: chunk bits (physical) shared by the sweep before and the
    # sweep after, so both can run in 2^len(cbits) parts pipelined with the remap
    cbits: list = field(default_factory=list)
    pre: int = -1  # descriptor of the sweep before the remap
    post: int = -1  # descriptor of the sweep after the remap
    # sweeps before the remap that run depth-first in parts (oldest first,
    # ending with `pre`): chunk c of all of them, then chunk c of the remap
    chain: list = field(default_factory=list)
    # localize: the next sweep reads region alpha through a load XOR (no region move)
    folded: bool = False


@dataclass
class DeviceProgram:
    buf: "ProgramBuffers"
    steps: list
    init_perm: list  # reference device bit -> physical device bit at Alloc
    n_fused: int
    # ApplyFused slot -> slot whose sweep measured its norm (itself, a later
    # slot when leaves share a sweep, an earlier one after trailing
    # relabels); slots absent here precede every sweep and carry the
    # initial norm
    norm_alias: dict = field(default_factory=dict)


class _Lookahead:
    """Future needs of the remaining primitive stream, in current reference labels."""

    def __init__(self, stream: list, start: int, n_local: int):
        lab = list(range(max(n_local, 1) + 64))
        first_use: dict = {}
        self.exchange: list = []  # current labels of the next remap's local bits
        for i in range(start, len(stream)):
            pr = stream[i]
            if isinstance(pr, Swap):
                lab[pr.a], lab[pr.b] = lab[pr.b], lab[pr.a]
            elif isinstance(pr, ExchMark):
                if not self.exchange:
                    self.exchange = [lab[b] for b in pr.bits]
            else:
                for b in _needs(pr):
                    cur = lab[b]
                    if cur not in first_use:
                        first_use[cur] = i
        self.first_use = first_use
        # at the end reference label y must sit at physical y; label y then is
        # the data that now carries label lab[y]
        self.home = {lab[y]: y for y in range(len(lab))}


def _choose_store(tile: list, where: list, look: _Lookahead, low: int, n_local: int) -> dict:
    """Store permutation within the tile: physical tile bit -> destination bit."""
    inv = {p: r for r, p in enumerate(where[:n_local])}
    ids = [inv[p] for p in tile if p in inv]  # reference labels living in the tile
    fixed = [p for p in tile if p not in inv]  # row / phantom bits stay put
    dest = {p: p for p in fixed}
    free = set(p for p in tile if p in inv)
    placed: dict = {}
    # qubits of the next remap go to the top physical bits first: contiguous
    # regions, so the NCCL exchange needs no pack/unpack pass
    tops = [p for p in range(n_local - 1, n_local - 1 - len(look.exchange), -1) if p in free]
    for r in look.exchange:
        if r in ids and tops:
            placed[r] = tops.pop(0)
            free.discard(placed[r])
    lows = [p for p in range(low) if p in free]
    soon = sorted((r for r in ids if r in look.first_use and r not in placed),
                  key=lambda r: look.first_use[r])
    for p, r in zip(lows, soon):
        placed[r] = p
    free -= set(placed.values())
    for r in ids:
        if r in placed:
            continue
        h = look.home.get(r, r)
        if h in free:
            placed[r] = h
            free.discard(h)
    for r in ids:  # the rest keep their place when possible
        if r not in placed and where[r] in free:
            placed[r] = where[r]
            free.discard(where[r])
    rest = sorted(free)
    for r in ids:
        if r not in placed:
            placed[r] = rest.pop(0)
    for r, p_new in placed.items():
        dest[where[r]] = p_new
    return dest


def _pad_displaced(tile: set, where: list, look: _Lookahead, K: int, L: int) -> None:
    """Fill free tile slots with (position, home) pairs of displaced qubits."""
    for r in range(L):
        if len(tile) >= K:
            return
        h = look.home.get(r, r)
        if h >= L or where[r] == h:
            continue
        add = {where[r], h} - tile
        if len(tile) + len(add) <= K:
            tile |= add


# sweeps may span consecutive ApplyFused leaves (plan_device.run_segment)
MERGE_LEAVES = os.environ.get("SVB200_MERGE_LEAVES", "1") not in ("0", "false", "no")
MAX_CHAIN = int(os.environ.get("SVB200_MAX_CHAIN", "3"))  # sweeps before a remap run depth-first with it
# chunk bits and swapped bits of an overlapped remap stay at or above this
# physical bit: the bulk-copy swap moves contiguous runs of 2^bit amplitudes
# and needs >= 4 KB pieces to keep NVLink busy (tools/p2p_bench.py)
MIN_OVERLAP_BIT = 8


def _plan_overlap(steps: list, buf, geo: DeviceGeometry, nbits: int, max_chain: int = MAX_CHAIN,
                  skip_first: bool = False) -> None:
    """Chunk bits for remaps whose neighbouring sweeps can run in parts.

    The chunk bits lie outside the tiles of the sweep after the remap, of a
    chain of up to `max_chain` sweeps before it and of the swapped bits, so
    every part touches one chunk only: chunk c of the chain, the remap of
    chunk c and chunk c of the sweep after form one pipeline stage."""
    if nbits <= 0:
        return
    L = geo.L + geo.h  # planner-owned bits (local + rows of this device)
    first_seen = False
    for i, st in enumerate(steps):
        if st.kind != "exchange" or not st.swaps:
            continue
        if skip_first and not first_seen:  # its sweeps run sparse (sparse_start) instead
            first_seen = True
            continue
        first_seen = True
        if any(ib < geo.h for ib, _ in st.swaps):
            continue  # part of the remap is an in-HBM bit swap over all chunks
        if min(lb for _, lb in st.swaps) < MIN_OVERLAP_BIT:
            continue  # short runs: the swap needs the whole GPU (register kernel)
        # sweeps on each side, nearest first; relabel-only leaves move no data
        before = []
        for x in reversed(steps[:i]):
            if x.kind in ("exchange", "localize"):  # a replicated sparse prefix stays whole
                break
            before.extend(range(x.first + x.count - 1, x.first - 1, -1))
        nxt = None
        for x in steps[i + 1:]:
            if x.kind == "exchange":
                break
            if x.count:
                nxt = x
                break
        if not before or nxt is None:
            continue
        post = nxt.first
        if buf.descs[post].get("cbits"):
            continue
        busy = set(buf.descs[post]["tin"]) | {lb for _, lb in st.swaps}
        have = buf.descs[before[0]].get("cbits")  # pre is also the post of an earlier remap
        if have:
            if busy & set(have) or set(buf.descs[before[0]]["tin"]) & set(have):
                continue
            chain, cb = [before[0]], list(have)
        else:
            chain, cb = [], None
            for di in before[:max_chain]:
                if buf.descs[di].get("cbits") or di == 0:
                    break  # chunked for an earlier remap / may synthesise |0...0>
                trial = busy | set(buf.descs[di]["tin"])
                cand = [b for b in range(L - 1, MIN_OVERLAP_BIT - 1, -1) if b not in trial]
                if len(cand) < nbits:
                    break
                chain.append(di)
                busy = trial
                cb = sorted(cand[:nbits])
            if not chain:
                continue
        st.cbits, st.pre, st.post = cb, chain[0], post
        st.chain = list(reversed(chain))
        for di in chain:
            buf.descs[di]["cbits"] = cb
        buf.descs[post]["cbits"] = cb


def plan_device(plan, geo: DeviceGeometry, kmax: int = KMAX, low: int = LOW_RUN_BITS,
                max_materialize: int = 64, rb: int = RB, fuse: bool = True,
                overlap_bits: int = 0, free_start: bool = True, stable_threads: bool = False,
                overlap_skip_first: bool = False, replicate_prefix: bool = False) -> DeviceProgram:
    """Compile every ApplyFused task of a plan for one device, with a global layout.

    The physical layout is a permutation `where` of the local bits that the
    planner owns: SWAP gates only relabel, every sweep stores its tile with a
    permutation that parks the next sweep's qubits on the low (contiguous)
    bits and moves other qubits toward their final position, and trailing
    materialization sweeps restore the reference layout before the state is
    returned.  The schedule depends only on the plan structure, so every
    device of a distributed run derives the same layouts.

    free_start: the run starts from |0...0> (invariant under any layout), so
    the planner may pick the initial physical layout; otherwise it starts
    from the reference layout and an initial state loads with no permutation.
    """
    L, D = geo.L, geo.D
    K = min(kmax, D)
    low = min(low, K)
    # replicate_prefix (run from |0...0>, see localize_applies): every
    # process computes the sweeps before the first remap as the process that
    # holds the unit amplitude, and that remap becomes a local region move
    first_remote = None
    if replicate_prefix:
        for ti, task in enumerate(plan.tasks):
            if task.kind == "Exchange" and any(geo.g - 1 - sw["rank_bit"] >= geo.h for sw in task.payload["swaps"]):
                first_remote = ti
                break
    geo0 = DeviceGeometry(d=geo.d, g=geo.g, h=geo.h, rank_base=0, pad_to=geo.pad_to)
    prefix_ids = set()
    raw = {}
    for ti, task in enumerate(plan.tasks):
        if task.kind == "ApplyFused":
            layout = plan.layout_phases[task.payload["phase"]]
            in_prefix = first_remote is not None and ti < first_remote
            if in_prefix:
                prefix_ids.add(task.id)
            prims = []
            for e in task.payload["gates"]:
                prims.extend(resolve_entry(e, layout, geo0 if in_prefix else geo))
            raw[task.id] = prims
    # segments: runs of ApplyFused tasks with no remap between them.  With
    # MERGE_LEAVES the gate fusion runs over a whole segment (an SU(4) split
    # between two leaves is fused again); each fused primitive belongs to the
    # latest task it contains a gate of
    segs, cur = [], []
    for task in plan.tasks:
        if task.kind == "ApplyFused":
            cur.append(task)
        elif task.kind == "Exchange" and cur:
            segs.append(cur)
            cur = []
    if cur:
        segs.append(cur)
    seg_prims = {}  # first task id -> (prims, owners)
    for seg in segs:
        prims, owners = [], []
        if MERGE_LEAVES and fuse:
            for ti, task in enumerate(seg):
                prims.extend(raw[task.id])
                owners.extend([ti] * len(raw[task.id]))
            prims, owners = fuse_prims(prims, owners)
        else:
            for ti, task in enumerate(seg):
                ps = fuse_prims(raw[task.id]) if fuse else raw[task.id]
                prims.extend(ps)
                owners.extend([ti] * len(ps))
        seg_prims[seg[0].id] = (prims, owners)
    # planning stream: every segment's primitives, with a marker per remap
    stream, leaf_start = [], {}
    for task in plan.tasks:
        if task.kind == "ApplyFused":
            if task.id in seg_prims:
                leaf_start[task.id] = len(stream)
                stream.extend(seg_prims[task.id][0])
        elif task.kind == "Exchange":
            remote_bits = []
            for s in task.payload["swaps"]:
                ib = geo.g - 1 - s["rank_bit"]
                if ib < geo.h:  # rank bit held by this device: a relabel (see below)
                    stream.append(Swap(L + ib, L - 1 - s["local_bit"]))
                else:
                    remote_bits.append(L - 1 - s["local_bit"])
            stream.append(ExchMark(tuple(remote_bits)))

    buf = ProgramBuffers()
    steps: list = []
    where = list(range(D))
    # bits the planner owns: the local bits and the rank bits held as rows on
    # this device (phantom pad bits stay put); a remap between a row bit and a
    # local bit only relabels them
    NL = L + geo.h
    # the |0...0> start is layout-invariant: pick the first layout like a store
    init = list(where)
    if free_start:
        look0 = _Lookahead(stream, 0, NL)
        d0 = _choose_store(list(range(NL)), where, look0, low, NL)
        for r in range(NL):
            init[r] = d0[where[r]]
    where = list(init)

    norm_alias: dict = {}
    last_measured = -1  # slot of the latest sweep-measured norm
    task_slot = {}
    for task in plan.tasks:
        if task.kind == "ApplyFused":
            task_slot[task.id] = len(task_slot)

    def run_segment(seg: list) -> None:
        """Sweeps for a run of consecutive ApplyFused tasks (no remap between
        them).  With MERGE_LEAVES a sweep may span several leaves: gates of
        consecutive leaves share a tile whenever their qubits fit, so the
        many small leaves the partitioner emits (one to three gates on one
        or two qubits) cost no memory pass of their own.  Each sweep is
        launched by the task it ends in; a leaf that ends inside a sweep
        takes that sweep's norm (gates are unitary: the norm after the
        sweep is the norm after the leaf, up to rounding)."""
        nonlocal last_measured
        prims, owner = seg_prims[seg[0].id]
        # task t is complete once every primitive owned by tasks <= t is
        # emitted: ends[t] = 1 + last such position
        last = {}
        for k, o in enumerate(owner):
            last[o] = k + 1
        ends, e = [], 0
        for ti in range(len(seg)):
            e = max(e, last.get(ti, 0))
            ends.append(e)
        n = len(prims)
        base = leaf_start[seg[0].id]
        firsts = {ti: None for ti in range(len(seg))}
        counts = {ti: 0 for ti in range(len(seg))}
        completed = 0  # tasks [0, completed) are done
        i = 0
        # tasks with no primitives before the first sweep carry the previous norm
        while completed < len(seg) and ends[completed] == 0:
            completed += 1
        while i < n:
            limit = n if MERGE_LEAVES else min(e for e in ends if e > i)
            if all(isinstance(pr, Swap) for pr in prims[i:limit]):
                # relabels only (the rest of the segment, or a SWAP-only
                # leaf when leaves are not merged): no data moves
                for pr in prims[i:limit]:
                    where[pr.a], where[pr.b] = where[pr.b], where[pr.a]
                i = limit
                while completed < len(seg) and ends[completed] <= i:
                    if last_measured >= 0:
                        norm_alias[task_slot[seg[completed].id]] = last_measured
                    completed += 1
                continue
            # greedy extent of this sweep under the current layout
            trial = list(where)
            need = set(range(low))
            j = i
            while j < limit:
                pr = prims[j]
                if isinstance(pr, Swap):
                    trial[pr.a], trial[pr.b] = trial[pr.b], trial[pr.a]
                    j += 1
                    continue
                nb = {trial[b] for b in _needs(pr)}
                if len(need | nb) > K and j > i:
                    break
                need |= nb
                j += 1
            # pad the tile with the next qubits needed after this sweep so the
            # store can park them on the low bits
            look = _Lookahead(stream, base + j, NL)
            tile = set(need)

            def park_exchange():  # let the store park the next remap's qubits on top
                for r in look.exchange:
                    if len(tile) + 2 <= K:
                        tile.add(trial[r])
                for p_top in range(NL - 1, NL - 1 - len(look.exchange), -1):
                    if len(tile) < K:
                        tile.add(p_top)

            # the sweep that ends the segment reserves room for that first: no
            # gate may need the remap's qubits (phase-only blocks), and the
            # next-needed padding would otherwise fill the tile
            before_remap = j >= n and bool(look.exchange) and PARK_FIRST
            if before_remap:
                park_exchange()
            for r in sorted(look.first_use, key=look.first_use.get):
                if len(tile) >= K:
                    break
                tile.add(trial[r])
            if not before_remap:
                park_exchange()
            _pad_displaced(tile, trial, look, K, NL)
            for b in range(D):
                if len(tile) >= K:
                    break
                tile.add(b)
            tile = sorted(tile)
            sp = build_sweep(prims[i:j], tile, where)  # updates `where` (swaps)
            dest = _choose_store(tile, where, look, low, NL)
            inv = {p: r for r, p in enumerate(where[:NL])}
            for p in tile:
                _, fl = sp.out_map[p]
                sp.out_map[p] = (dest[p], fl)
            for p in tile:
                if p in inv:
                    where[inv[p]] = dest[p]
            done = []
            while completed < len(seg) and ends[completed] <= j:
                done.append(task_slot[seg[completed].id])
                completed += 1
            sp.norm_slot = done[-1] if done else -1
            if seg[0].id in prefix_ids and geo.rank_base != 0:
                sp.norm_slot = -1  # a replica of process 0's prefix: its norm counts once
            for sl in done:
                norm_alias[sl] = done[-1]
            if done:
                last_measured = done[-1]
            at = min(t for t, e in enumerate(ends) if e >= j)  # launched by the task it ends in
            if firsts[at] is None:
                firsts[at] = len(buf.descs)
            counts[at] += 1
            emit_sweep(sp, geo, buf, rb, stable_threads)
            i = j
        for ti, task in enumerate(seg):
            f = firsts[ti] if firsts[ti] is not None else len(buf.descs)
            steps.append(Step("sweeps", task.id, f, counts[ti]))

    seg: list = []
    for task in plan.tasks:
        if task.kind == "ApplyFused":
            seg.append(task)
            continue
        if task.kind != "Exchange":
            continue
        if seg:
            run_segment(seg)
            seg = []
        sw = []
        for s in task.payload["swaps"]:
            ib = geo.g - 1 - s["rank_bit"]
            lb = L - 1 - s["local_bit"]
            if ib < geo.h:  # executor.py:224-281 moves data between rows of this
                # device: here only the labels of the two bits swap
                where[L + ib], where[lb] = where[lb], where[L + ib]
            else:
                sw.append((ib, where[lb]))
        # the first remote remap after a replicated prefix moves no data
        # between GPUs (localize_applies): each process keeps its region
        kind = "localize" if (first_remote is not None and plan.tasks.index(task) == first_remote) else "exchange"
        steps.append(Step(kind, task.id, swaps=sw))
    if seg:
        run_segment(seg)
    slot = len(task_slot)

    _plan_overlap(steps, buf, geo, overlap_bits, skip_first=overlap_skip_first)

    # restore the reference layout
    first = len(buf.descs)
    passes = 0
    while any(where[r] != r for r in range(NL)):
        if passes >= max_materialize:
            raise RuntimeError("layout materialization did not converge")
        passes += 1
        tile = set(range(low))
        for r in range(NL):
            if len(tile) + 2 > K:
                break
            if where[r] != r and (where[r] not in tile or r not in tile):
                cand = tile | {where[r], r}
                if len(cand) <= K:
                    tile = cand
        for b in range(D):
            if len(tile) >= K:
                break
            tile.add(b)
        tile = sorted(tile)
        look = _Lookahead([], 0, NL)
        sp = build_sweep([], tile, where)
        dest = _choose_store(tile, where, look, 0, NL)
        inv = {p: r for r, p in enumerate(where[:NL])}
        for p in tile:
            sp.out_map[p] = (dest[p], 0)
        for p in tile:
            if p in inv:
                where[inv[p]] = dest[p]
        emit_sweep(sp, geo, buf, rb, stable_threads)
    if passes:
        steps.append(Step("materialize", None, first, passes))
    return DeviceProgram(buf=buf, steps=steps, init_perm=init, n_fused=slot, norm_alias=norm_alias)


def sparse_start(dp: "DeviceProgram", D: int, unit: bool) -> dict:
    """Support of the state along the sweeps of a run that starts from |0...0>.

    A sweep changes amplitudes only along its tile bits, and its store
    permutes the tile bits among themselves, so from |0...0> the amplitudes
    that can be nonzero are those whose physical bits outside a support set
    S are 0, with S growing by each sweep's tile bits (S starts empty with
    the unit amplitude at index 0 of the device holding it, or None on the
    devices that hold only zeros).  Returns {descriptor: (S_in, full_out)}
    for the leading sweeps whose S_in is not the whole device: they compute
    only the tiles inside the support (jit.kernel_source) and the last one
    also writes the zeros outside it (full_out), after which the state is
    fully materialised.  The sequence ends at the first remap that moves
    data, at a sweep that runs in parts around an overlapped remap, or when
    the support covers every bit.  The first sweep must have a register
    stage to synthesise the unit vector; otherwise no sweep is sparse."""
    full = (1 << D) - 1
    supp = 0 if unit else None
    seq = []
    stop = False
    for st in dp.steps:
        if stop:
            break
        if st.kind == "localize":
            # the region of this process moved to region 0 of the swapped
            # bits; the other regions hold stale prefix data, read as zeros
            if supp is not None:
                supp &= ~sum(1 << lb for _, lb in st.swaps)
            continue
        if st.kind == "exchange":
            if st.swaps:
                break
            continue  # a relabel: no data moves
        for i in range(st.first, st.first + st.count):
            d = dp.buf.descs[i]
            if d.get("cbits") or (supp is not None and supp == full):
                stop = True
                break
            seq.append((i, supp))
            if supp is not None:
                tin = [int(b) for b in d["tin"][:d["K"]]]
                assert sorted(tin) == sorted(int(b) for b in d["st_dev"][:d["K"]]), "store leaves the tile"
                supp |= sum(1 << b for b in tin)
    if not seq:
        return {}
    i0, s0 = seq[0]
    d0 = dp.buf.descs[i0]
    ops = dp.buf.ops[d0["op_begin"]: d0["op_begin"] + d0["op_count"]]
    if s0 == 0 and not any(int(o["kind"]) == OP_STAGE for o in ops):
        return {}
    return {i: (s, k == len(seq) - 1) for k, (i, s) in enumerate(seq)}


def localize_applies(dp: "DeviceProgram", D: int, world: int, h: int) -> bool:
    """From |0...0> every sweep before the first inter-process remap is sparse
    (cheap), and that remap swaps every process-id bit.  Then after the remap
    process w holds exactly region alpha_w (its id bits) of the state that
    the process holding the unit amplitude had before it, moved to region 0
    of the swapped local bits, and zeros elsewhere: every process can compute
    that prefix itself (a replica, a fraction of a pass) and move its region
    locally, so no amplitude crosses NVLink for that remap."""
    if world < 2 or not sparse_reaches_first_remap(dp, D):
        return False
    for st in dp.steps:
        if st.kind == "exchange" and st.swaps:
            ids = {ib - h for ib, _ in st.swaps if ib >= h}
            return ids == set(range(world.bit_length() - 1))
    return False


def sparse_reaches_first_remap(dp: "DeviceProgram", D: int) -> bool:
    """True when, from |0...0> on the device holding the unit vector, every
    sweep before the first data-moving remap is sparse (its support never
    covers the device): those sweeps then cost a fraction of a pass, and
    running them in overlapped parts (which keeps them dense) would be
    slower than the remap they hide behind.  Decided on a program planned
    without overlap, identically on every process."""
    sp = sparse_start(dp, D, True)
    for st in dp.steps:
        if st.kind == "exchange" and st.swaps:
            return True
        if st.kind in ("sweeps", "materialize"):
            if any(i not in sp for i in range(st.first, st.first + st.count)):
                return False
    return False


def sparse_bytes(desc: dict, sparse) -> tuple:
    """(bytes read, bytes written) of one sweep launch: 16 B per amplitude;
    a sparse sweep reads only the support and writes only live tiles (plus
    every dead position when full_out)."""
    K, D = int(desc["K"]), int(desc["D"])
    if sparse is None:
        return 16 << D, 16 << D
    supp, full_out = sparse
    if supp is None:
        return 0, (16 << D) if full_out else 0
    tinm = sum(1 << int(b) for b in desc["tin"][:K])
    nsupp = bin(supp).count("1")
    nlive_fixed = bin(supp & ~tinm).count("1")
    rd = 0 if supp == 0 else 16 << nsupp
    wr = (16 << D) if full_out else 16 << (nlive_fixed + K)
    return rd, wr


def _independent3(vs) -> bool:
    a, b, c = vs
    return all(x != 0 for x in (a, b, c, a ^ b, a ^ c, b ^ c, a ^ b ^ c))


def _choose_swizzle(K: int, patterns: list, seed: int = 0) -> list:
    """Per-tile-bit smem images so every access pattern is bank-conflict free.

    A 16-byte access by 8 lanes is conflict free iff the lanes' addresses
    differ in the low 3 bits of the (16 B-unit) smem index; each pattern lists
    the 3 tile bits that vary across a quarter warp.
    """
    low = [1 << k if k < 3 else 0 for k in range(K)]

    def ok(lows):
        return all(_independent3([lows[k] for k in pat]) for pat in patterns if len(pat) == 3)

    base = [(1 << k) if k < 3 else (1 << (k % 3)) for k in range(K)]
    if ok(base):
        lows = base
    else:
        rng = np.random.default_rng(seed)
        lows = None
        for _ in range(4000):
            cand = [(1 << k) if k < 3 else int(rng.integers(0, 8)) for k in range(K)]
            if ok(cand):
                lows = cand
                break
        if lows is None:
            lows = base  # correct, only slower
    del low
    return [(1 << k) if k < 3 else ((1 << k) | lows[k]) for k in range(K)]


def _thread_orders(stages: list, K: int, stable: bool) -> list:
    """Tile bit held by each thread bit, per stage.

    Default: ascending tile bits.  `stable` (generated kernels): a tile bit
    that stays a thread bit keeps its thread-bit position, and the warp-level
    positions (thread bits >= 5) hold the bits needed last; a stage change
    that then leaves the warp bits in place moves data within warps only
    (warp shuffles, no shared memory or barrier; jit.kernel_source)."""
    n = len(stages)

    def next_use(k, si):
        for sj in range(si + 1, n):
            if k in stages[sj][0]:
                return sj
        return n + 1

    orders, prev = [], None
    for si, (rbits_s, _) in enumerate(stages):
        tb = [k for k in range(K) if k not in rbits_s]
        if not stable:
            order = tb
        elif prev is None:
            order = sorted(tb, key=lambda k: (next_use(k, si), k))
        else:
            order = list(prev)
            vacated = sorted((p for p, k in enumerate(prev) if k in rbits_s), reverse=True)
            incoming = sorted((k for k in tb if k not in prev), key=lambda k: (-next_use(k, si), k))
            for p, k in zip(vacated, incoming):
                order[p] = k
        orders.append(order)
        prev = order
    return orders


def pack_order(order: list) -> int:
    v = 0
    for i, k in enumerate(order):
        v |= int(k) << (4 * i)
    return v


def unpack_order(val: int, n: int) -> list:
    return [(int(val) >> (4 * i)) & 15 for i in range(n)]


STAGE_SCHED = os.environ.get("SVB200_STAGE_SCHED", "1") not in ("0", "false", "no")


def _touched(it, tin: list) -> set:
    """Physical device bits an item reads or writes (targets, controls, phases)."""
    out = {tin[k] for k in it.bits}
    out |= set(it.ctrl)
    for f in it.factors:
        out |= set(f.bits)
    return out


def _stages_sched(items: list, rb: int, tin: list) -> list:
    """Stages by list scheduling: items that touch disjoint bits commute, so
    a stage may take any item whose predecessors on its bits are scheduled
    and whose register bits fit the stage.  Each stage starts from the ready
    item that lets the most items join it.  Fewer stages = fewer shared-
    memory round trips per tile (a stage moves the whole 64 KB tile)."""
    n = len(items)
    touched = [_touched(it, tin) for it in items]
    preds = [set() for _ in range(n)]
    last: dict = {}
    for i in range(n):
        for b in touched[i]:
            if b in last:
                preds[i].add(last[b])
        for b in touched[i]:
            last[b] = i
    done = [False] * n
    left = n
    stages = []

    def grow(seed_bits: set, seed_order: list) -> tuple:
        need, order = set(seed_bits), list(seed_order)
        taken = set(order)
        while True:  # add the fitting ready item that needs the fewest new register bits
            pick, cost = None, None
            for i in range(n):
                if done[i] or i in taken or not all(done[p] or p in taken for p in preds[i]):
                    continue
                nb = set(items[i].bits)
                if len(need | nb) > rb:
                    continue
                c = len(nb - need)
                if cost is None or c < cost:
                    pick, cost = i, c
                    if c == 0:
                        break
            if pick is None:
                return need, order
            need |= set(items[pick].bits)
            order.append(pick)
            taken.add(pick)

    while left:
        ready = [i for i in range(n) if not done[i] and all(done[p] for p in preds[i])]
        best = None
        for r in ready[:24]:  # seeds: the first ready items (bounded work per stage)
            need, order = grow(set(items[r].bits), [r])
            if best is None or len(order) > len(best[1]):
                best = (need, order)
        need, order = best
        order.sort()  # program order inside the stage (dependencies hold)
        for i in order:
            done[i] = True
        left -= len(order)
        stages.append([need, [items[i] for i in order]])
    return stages


def _stages(items: list, rb: int = RB) -> list:
    """Group items into stages of <= rb register bits; returns [(rbits, items)]."""
    stages = []
    cur, need = [], set()
    for it in items:
        nb = set(it.bits)
        if len(need | nb) > rb and cur:
            stages.append([need, cur])
            cur, need = [], set()
        cur.append(it)
        need |= nb
    if cur:
        stages.append([need, cur])
    return stages


@dataclass
class ProgramBuffers:
    ops: list = field(default_factory=list)  # dicts -> OP_DTYPE
    coef: list = field(default_factory=list)  # complex
    tab: list = field(default_factory=list)  # np arrays (complex)
    tab_len: int = 0
    cterms: list = field(default_factory=list)  # (dst, mask, c) per sweep
    cofs: list = field(default_factory=list)  # int per sweep CSR
    descs: list = field(default_factory=list)

    def add_coef(self, vals) -> int:
        off = len(self.coef)
        self.coef.extend(complex(v) for v in vals)
        return off

    def add_tab(self, arr: np.ndarray) -> int:
        off = self.tab_len
        self.tab.append(np.asarray(arr, dtype=np.complex128))
        self.tab_len += len(arr)
        return off


def emit_sweep(sp: SweepProgram, geo: DeviceGeometry, buf: ProgramBuffers, rb: int = RB,
               stable: bool = False) -> None:
    K = sp.K
    tin = sp.tin
    dev_to_tile = {b: k for k, b in enumerate(tin)}
    NT = 1 << (K - rb)
    tidx = np.arange(NT, dtype=np.int64)

    items = list(sp.items)
    # fold the accumulated constant / H scale into the final phase item
    final = items[-1]
    assert final.kind == OP_PHALL
    body = [it for it in items if it.kind != OP_PHALL]
    stages = _stages_sched(body, rb, tin) if STAGE_SCHED else _stages(body, rb)
    if not stages and (final.factors or sp.scale != 1):
        stages = [[set(), []]]
    # pad register sets to exactly rb bits, preferring bits used soon after;
    # the last stage prefers bits that are not stored to output bits 0-4, so
    # those stay on lanes and the stage can store straight from registers
    # (jit.kernel_source direct stores)
    low_out = {k for k in range(K) if sp.out_map[tin[k]][0] < 5}
    for si, st in enumerate(stages):
        need = st[0]
        for later in stages[si + 1:]:
            for b in sorted(later[0]):
                if len(need) < rb and b not in need:
                    need.add(b)
        last = si == len(stages) - 1 and len(stages) >= 2  # one-stage sweeps keep the smem store path
        fill = sorted(range(K), key=lambda b: (b in low_out, b)) if last else range(K)
        for b in fill:
            if len(need) >= rb:
                break
            need.add(b)
        st[0] = need
    if stages:
        # leftover factors: anchor those touching a last-stage register bit on
        # that bit (OP_PH), the rest become one thread-uniform OP_PHALL
        last_r = stages[-1][0]
        by_anchor: dict = {}
        rest_f = []
        for f in final.factors:
            ks = [dev_to_tile.get(b) for b in f.bits]
            regs = [k for k in ks if k is not None and k in last_r]
            if regs:
                by_anchor.setdefault(min(regs), []).append(f)
            else:
                rest_f.append(f)
        for k in sorted(by_anchor):
            stages[-1][1].append(_Item(OP_PH, (k,), factors=by_anchor[k]))
        stages[-1][1].append(_Item(OP_PHALL, (), factors=rest_f))

    # smem swizzle: load (tile bits 0..2), store order, each stage's thread bits
    store_order = sorted(range(K), key=lambda k: sp.out_map[tin[k]][0])
    patterns = [[0, 1, 2], store_order[:3]]
    orders = _thread_orders(stages, K, stable)
    for comp in orders:
        patterns.append(comp[:3])
    sw = _choose_swizzle(K, [p for p in patterns if len(p) == 3])

    ctab_terms: dict = {}  # slot -> list of (mask, c)
    nct = [0]

    def new_ctab() -> int:
        s = nct[0]
        nct[0] += 1
        ctab_terms[s] = []
        return s

    op_begin = len(buf.ops)
    for (rbits, sitems), comp in zip(stages, orders):
        rlist = sorted(rbits)
        slot_of = {k: i for i, k in enumerate(rlist)}
        tbit_of = {k: i for i, k in enumerate(comp)}
        rmask = 0
        for k in rlist:
            rmask |= 1 << k
        if stable:
            buf.ops.append(dict(kind=OP_STAGE, rmask=rmask, flags=F_TORDER, pval=pack_order(comp)))
        else:
            buf.ops.append(dict(kind=OP_STAGE, rmask=rmask))
        for it in sitems:
            op = dict(kind=it.kind, a=0, b=0, rmask=0, pmask=0, pval=0, coef=0, tab=-1,
                      ctab=-1, tf=-1, flags=0)
            if it.bits:
                op["a"] = slot_of[it.bits[0]]
            # controls: register bits -> rmask (slot mask); others -> predicate
            for cb, val in it.ctrl.items():
                k = dev_to_tile.get(cb)
                if k is not None and k in slot_of:
                    op["rmask"] |= 1 << slot_of[k]
                    op["b"] |= val << slot_of[k]
                else:
                    op["pmask"] |= 1 << cb
                    op["pval"] |= val << cb
            # phase factors -> (const, per-thread table, per-tile slots, register factors)
            pre_const = complex(1.0)
            preg = [complex(1.0)] * rb
            tab = None
            tf_terms: dict = {}
            scal_terms: list = []
            anchor = it.bits[0] if it.bits else None
            for f in it.factors:
                rest = [b for b in f.bits if not (anchor is not None and dev_to_tile.get(b) == anchor)]
                if anchor is not None and len(rest) == len(f.bits):
                    raise AssertionError("flushed factor does not touch its anchor bit")
                if not rest:
                    pre_const *= f.c
                    continue
                if len(rest) == 1:
                    b = rest[0]
                    k = dev_to_tile.get(b)
                    if k is not None and k in slot_of:
                        if anchor is None:
                            raise AssertionError("register factor without anchor")
                        preg[slot_of[k]] *= f.c
                    elif k is not None:
                        if tab is None:
                            tab = np.ones(NT, dtype=np.complex128)
                        tab[((tidx >> tbit_of[k]) & 1) == 1] *= f.c
                    else:
                        scal_terms.append((1 << b, f.c))
                    continue
                # two bits, no anchor (final PHALL / PH item)
                b0, b1 = rest
                k0, k1 = dev_to_tile.get(b0), dev_to_tile.get(b1)
                in0 = k0 is not None and k0 in slot_of
                in1 = k1 is not None and k1 in slot_of
                if in0 or in1:
                    raise AssertionError("register factor reached PHALL")
                if k0 is not None and k1 is not None:
                    if tab is None:
                        tab = np.ones(NT, dtype=np.complex128)
                    sel = (((tidx >> tbit_of[k0]) & 1) == 1) & (((tidx >> tbit_of[k1]) & 1) == 1)
                    tab[sel] *= f.c
                elif k0 is None and k1 is None:
                    scal_terms.append(((1 << b0) | (1 << b1), f.c))
                else:
                    kt, bf = (k0, b1) if k0 is not None else (k1, b0)
                    tf_terms.setdefault(tbit_of[kt], []).append((1 << bf, f.c))
            if it.kind == OP_PHALL:
                pre_const *= sp.scale
            has_phase = bool(it.factors) or it.kind == OP_PHALL
            if it.kind in (OP_PH, OP_H, OP_U1) and it.factors:
                if it.kind != OP_PH and (op["pmask"] or (it.kind == OP_H and op["rmask"])):
                    raise AssertionError("pre-phase on a predicated gate")
                op["flags"] |= F_PHASE
            if has_phase:
                if scal_terms:
                    s = new_ctab()
                    ctab_terms[s].extend(scal_terms)
                    op["ctab"] = s
                if tf_terms:
                    first = None
                    for i in range(K - rb):
                        s = new_ctab()
                        if first is None:
                            first = s
                        ctab_terms[s].extend(tf_terms.get(i, []))
                    op["tf"] = first
                if tab is not None:
                    op["tab"] = buf.add_tab(tab)
                nt = 0
                for i in range(rb):
                    if preg[i] != 1:
                        nt |= 1 << i
                op["flags"] |= nt << F_PREG_SHIFT
            if it.kind == OP_PHALL:
                if not has_phase:
                    continue
                if op["ctab"] < 0 and op["tab"] < 0 and op["tf"] < 0:
                    if pre_const == 1:
                        continue
                    op["kind"] = OP_SCALE
                op["coef"] = buf.add_coef([pre_const])
            elif it.kind == OP_PH:
                op["coef"] = buf.add_coef([pre_const] + preg)
            elif it.kind in (OP_H, OP_U1):
                m = it.m if it.m is not None else np.eye(2)
                op["coef"] = buf.add_coef([m[0, 0], m[0, 1], m[1, 0], m[1, 1], pre_const] + preg)
            elif it.kind == OP_X:
                pass
            elif it.kind == OP_U2:
                a, b = slot_of[it.bits[0]], slot_of[it.bits[1]]
                mm = np.asarray(it.m)
                if a > b:  # kernel wants a < b with a as the matrix MSB
                    perm = [0, 2, 1, 3]
                    mm = mm[np.ix_(perm, perm)]
                    a, b = b, a
                op["a"], op["b"] = a, b
                op["coef"] = buf.add_coef(mm.reshape(-1))
            buf.ops.append(op)
    op_count = len(buf.ops) - op_begin

    # per-tile term CSR for this sweep
    cofs_base = len(buf.cofs)
    terms_base = len(buf.cterms)
    offs = [terms_base]
    for s in range(nct[0]):
        for mask, c in ctab_terms[s]:
            buf.cterms.append((s, mask, c))
        offs.append(len(buf.cterms))
    buf.cofs.extend(offs)

    # the same terms as 8-bit lookup tables over the tile index (generated
    # kernels): slot s = prod_c LUT[s][c][(tile_id >> 8c) & 255], plus the
    # rare terms whose bits span two chunks
    fbits = [b for b in range(geo.D) if b not in dev_to_tile]
    fpos = {b: i for i, b in enumerate(fbits)}
    nch = max(1, (len(fbits) + 7) // 8)
    lut_off, residual = -1, []
    if nct[0]:
        lut = np.ones((nct[0], nch, 256), dtype=np.complex128)
        vals = np.arange(256)
        for s_ in range(nct[0]):
            res_s = []
            for mask, c in ctab_terms[s_]:
                idx = [fpos[b] for b in range(geo.D) if (mask >> b) & 1]
                chunks_ = {i // 8 for i in idx}
                if not idx:
                    lut[s_, 0, :] *= c
                elif len(chunks_) == 1:
                    k = chunks_.pop()
                    lm = sum(1 << (i - 8 * k) for i in idx)
                    lut[s_, k, (vals & lm) == lm] *= c
                else:
                    res_s.append((mask, c))
            residual.append(res_s)
        lut_off = buf.add_tab(lut.reshape(-1))

    tout = [sp.out_map[tin[k]][0] for k in range(K)]
    st_flip = 0
    for k in range(K):
        if sp.out_map[tin[k]][1]:
            st_flip |= 1 << tout[k]
    desc = dict(
        K=K, D=geo.D, tin=list(tin), sw=sw,
        st_dev=[tout[k] for k in store_order], st_sw=[sw[k] for k in store_order],
        st_flip=st_flip, op_begin=op_begin, op_count=op_count, nctab=nct[0],
        norm_slot=sp.norm_slot, cofs_index=cofs_base, rb=rb,
        lut_off=lut_off, lut_nch=nch, residual=residual,
    )
    buf.descs.append(desc)


def pack(buf: ProgramBuffers):
    """Serialize to (device blob bytes, descriptor array)."""
    ops = np.zeros(max(len(buf.ops), 1), dtype=OP_DTYPE)
    for i, o in enumerate(buf.ops):
        for k, v in o.items():
            ops[i][k] = v
    coef = np.array(buf.coef if buf.coef else [0j], dtype=np.complex128)
    tab = np.concatenate(buf.tab) if buf.tab else np.zeros(1, dtype=np.complex128)
    ct = np.zeros(max(len(buf.cterms), 1), dtype=CTERM_DTYPE)
    for i, (dst, mask, c) in enumerate(buf.cterms):
        ct[i]["dst"] = dst
        ct[i]["mask"] = mask
        ct[i]["re"] = c.real
        ct[i]["im"] = c.imag
    cofs = np.array(buf.cofs if buf.cofs else [0], dtype=np.int32)

    parts = []
    off = 0

    def put(arr) -> int:
        nonlocal off
        b = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
        start = off
        parts.append(b)
        off += b.size
        pad = (-off) % 64
        if pad:
            parts.append(np.zeros(pad, dtype=np.uint8))
            off += pad
        return start

    ops_off = put(ops)
    coef_off = put(coef)
    tab_off = put(tab)
    ct_off = put(ct)
    cofs_off = put(cofs)
    blob = np.concatenate(parts) if parts else np.zeros(64, dtype=np.uint8)

    descs = np.zeros(len(buf.descs), dtype=DESC_DTYPE)
    for i, d in enumerate(buf.descs):
        e = descs[i]
        e["K"], e["D"] = d["K"], d["D"]
        for name in ("tin", "sw", "st_dev", "st_sw"):
            arr = np.zeros(MAXT, dtype=np.int32)
            arr[: len(d[name])] = d[name]
            e[name] = arr
        e["st_flip"] = d["st_flip"]
        e["op_begin"], e["op_count"] = d["op_begin"], d["op_count"]
        e["nctab"], e["norm_slot"] = d["nctab"], d["norm_slot"]
        e["rb"] = d.get("rb", RB)
        e["ops_off"], e["coef_off"], e["tab_off"] = ops_off, coef_off, tab_off
        e["cterm_off"] = ct_off
        e["cofs_off"] = cofs_off + 4 * d["cofs_index"]
    return blob, descs, dict(ops=ops, coef=coef, tab=tab, cterms=ct, cofs=cofs, cofs_base=cofs_off)
