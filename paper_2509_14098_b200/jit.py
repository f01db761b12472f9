"""Render compiled sweeps as straight-line CUDA and build them with NVRTC.

The generic sweep kernel (csrc/sweep.cu) interprets a short op list per
tile; on large states the interpretation overhead (op dispatch, register
moves between templated cases, runtime index math) dominates the FP64 work
(ncu: ~6,600 warp instructions per 4096-amplitude tile, ~1,550 of them
FP64).  Here each sweep becomes its own kernel: register slots, control
masks, smem swizzle offsets and gate coefficients are compile-time
constants, so what remains is the arithmetic plus one load and one store
per amplitude.  This is the reference paper's code-generation step (a
kernel per partition, section 4) performed at run time.

Kernels are compiled in parallel (NVRTC releases the GIL through ctypes)
and cached by source hash in memory and on disk.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

from . import _native
from . import program as prog

CSRC = Path(__file__).resolve().parent / "csrc"
CACHE_DIR = Path(os.environ.get("SVB200_JIT_CACHE", Path(__file__).resolve().parent.parent / "build" / "jit_cache"))
MAXREG_OVERLAP = int(os.environ.get("SVB200_JIT_MAXREG_OVERLAP", "232"))
# emit the ops before a stage and its shared-memory stores in two halves (see kernel_source)
SPLIT_STAGES = os.environ.get("SVB200_JIT_SPLIT", "0") not in ("0", "false", "no")  # measured: no gain
# per-tile slot tables of tile i+1 are loaded during tile i (off the tile-start critical path)
CTAB_AHEAD = os.environ.get("SVB200_JIT_CTAB_AHEAD", "1") not in ("0", "false", "no")
NO_AHEAD_ZERO = os.environ.get("SVB200_JIT_NO_AHEAD_ZERO", "1") not in ("0", "false", "no")
# stage changes that keep the warp-level thread bits move data with warp shuffles
SHUFFLE_STAGES = os.environ.get("SVB200_JIT_SHUFFLE", "0") not in ("0", "false", "no")  # measured: slower
# FP64-heavy sweeps can run two tile groups per CTA (kernel_source_2g,
# SVB200_JIT_GROUPS=1).  Off by default: QV-30 moved between -6% and +4%
# across boxes
GROUPS = os.environ.get("SVB200_JIT_GROUPS", "0") not in ("0", "false", "no")
NVRTC_OPTS = ["--gpu-architecture=sm_100a", "--std=c++17", f"-I{CSRC}", "-lineinfo",
              "--extra-device-vectorization"]



# ---------------------------------------------------------------------------
# expression helpers
# ---------------------------------------------------------------------------

def _lit_raw(x: float) -> str:
    r = repr(float(x))
    return r if ("e" in r or "." in r or "inf" in r or "nan" in r) else r + ".0"


# Coefficients of the kernel being generated can go to a __constant__ table
# (SVB200_JIT_CONST_POOL=1): FP64 literals are otherwise materialised with
# two UMOVs each (ncu round 2: 1,395 UMOVs beside 3,184 DFMAs per tile of the
# heaviest QV sweep).  Measured on B200: the table's uniform-register loads
# raise register pressure into spills and QV-30 ran 667 -> 731 ms, so it is off
_CONST_TABLE: dict | None = None
CONST_POOL = os.environ.get("SVB200_JIT_CONST_POOL", "0") not in ("0", "false", "no")
_INLINE = {0.0, 1.0, -1.0, 0.5, -0.5, 2.0, -2.0}


def _lit(x: float) -> str:
    x = float(x)
    if _CONST_TABLE is None or x in _INLINE or x != x:
        return _lit_raw(x)
    key = x.hex()
    i = _CONST_TABLE.setdefault(key, (len(_CONST_TABLE), x))[0]
    return f"kc[{i}]"


def _pool_begin() -> None:
    global _CONST_TABLE
    _CONST_TABLE = {} if CONST_POOL else None


def _pool_end(lines: list) -> list:
    """Insert the constant table after the include line."""
    global _CONST_TABLE
    pool, _CONST_TABLE = _CONST_TABLE, None
    if not pool:
        return lines
    vals = [v for _, v in sorted(pool.values())]
    decl = "__constant__ double kc[" + str(len(vals)) + "] = {" + ", ".join(_lit_raw(v) for v in vals) + "};"
    return lines[:1] + [decl] + lines[1:]


def _cmul_lit(expr: str, c: complex) -> str:
    cr, ci = float(c.real), float(c.imag)
    if ci == 0.0:
        if cr == 1.0:
            return expr
        if cr == -1.0:
            return f"make_double2(-({expr}).x, -({expr}).y)"
        return f"cmulr({expr}, {_lit(cr)})"
    if cr == 0.0:
        return f"make_double2(-({expr}).y * {_lit(ci)}, ({expr}).x * {_lit(ci)})"
    return f"cmulc({expr}, {_lit(cr)}, {_lit(ci)})"


# 4-term sums as two independent 2-term chains plus one add (shorter FP64
# dependency chains for one more DADD per component).  Measured on B200:
# QV-30 656 -> 703 ms, so it is off (SVB200_JIT_SPLIT_LINCOMB=1)
SPLIT_LINCOMB = os.environ.get("SVB200_JIT_SPLIT_LINCOMB", "0") not in ("0", "false", "no")


# real or imaginary coefficients accumulate with two FMAs (cfmar/cfmai)
REAL_IMAG_FMA = os.environ.get("SVB200_JIT_REAL_IMAG_FMA", "1") not in ("0", "false", "no")


def _lincomb(terms) -> str:
    """sum_k c_k * x_k for literal complex c_k (drops zero terms)."""
    terms = [(c, x) for c, x in terms if c != 0]
    if not terms:
        return "make_double2(0.0, 0.0)"
    if SPLIT_LINCOMB and len(terms) >= 4:
        h = len(terms) // 2
        return f"cadd({_lincomb_chain(terms[:h])}, {_lincomb_chain(terms[h:])})"
    return _lincomb_chain(terms)


def _lincomb_chain(terms) -> str:
    c0, x0 = terms[0]
    acc = _cmul_lit(x0, c0)
    for c, x in terms[1:]:
        cr, ci = float(c.real), float(c.imag)
        if ci == 0.0 and cr == 1.0:
            acc = f"cadd({acc}, {x})"
        elif ci == 0.0 and cr == -1.0:
            acc = f"csub({acc}, {x})"
        elif ci == 0.0 and REAL_IMAG_FMA:  # the dropped term is an exact zero
            acc = f"cfmar({x}, {_lit(cr)}, {acc})"
        elif cr == 0.0 and REAL_IMAG_FMA:
            acc = f"cfmai({x}, {_lit(ci)}, {acc})"
        else:
            acc = f"cfmac({x}, {_lit(cr)}, {_lit(ci)}, {acc})"
    return acc


def _deposit(var: str, dst_bits) -> str:
    """Expression placing bit i of `var` at position dst_bits[i] (runs merged)."""
    parts, i, n = [], 0, len(dst_bits)
    while i < n:
        j = i
        while j + 1 < n and dst_bits[j + 1] == dst_bits[j] + 1:
            j += 1
        width = j - i + 1
        mask = (1 << width) - 1
        shift = dst_bits[i]
        src = f"(((u64){var} >> {i}) & {mask}ull)"
        parts.append(f"({src} << {shift})" if shift > 0 else src)
        i = j + 1
    return " | ".join(parts) if parts else "0ull"


def _xor_img(var: str, imgs) -> str:
    parts = [f"((({var}) >> {i}) & 1u ? {int(s)}u : 0u)" for i, s in enumerate(imgs) if s]
    return " ^ ".join(parts) if parts else "0u"


# ---------------------------------------------------------------------------
# kernel generator
# ---------------------------------------------------------------------------

# stage changes that keep the warp-level thread bits (thread bits 5..) on the
# same tile bits move data only within each warp: a __syncwarp can replace
# the CTA barrier (planner-chosen stable thread-bit orders make 86 of QV-30's
# 163 stage changes warp-local).  Measured on B200: correct, but QV-30 ran
# 669 -> 691 ms (warps that drift apart in a ~200 KB straight-line kernel
# share fewer instruction fetches), so it is off by default
LOCAL_STAGES = os.environ.get("SVB200_JIT_LOCAL_STAGES", "0") not in ("0", "false", "no")


def _warp_local_change(stage_info: list, a: int, b: int, nthreads: int) -> bool:
    if not LOCAL_STAGES or nthreads < 64:
        return False
    return list(stage_info[a][1][5:]) == list(stage_info[b][1][5:])


def kernel_source(name: str, desc: dict, ops: list, coef: list, zero_init: int = 0,
                  sparse: tuple | None = None, ld_xor: int = 0, st_keep: tuple | None = None,
                  bcast: tuple | None = None) -> str:
    """Straight-line kernel for one sweep.

    bcast = (F mask, c, norm offset, slot): every value v is stored as c * v
    at its position P and at every P | f, f a combination of the F bits (the
    next sweep only expanded those dead bits; executor._broadcast_merges).
    Norms: sum |v|^2 at the launch's slot (offset None) or, for the merged
    sweep's leaf, 2^|F| sum |c v|^2 at the slot + offset (only that one when
    the offset is 0).

    st_keep = (mask, value): only positions whose tile bits at `mask` read
    `value` are stored (the last sweep of a replicated prefix: the localized
    remap keeps only this process's region).  The norm still covers every
    amplitude of the tile.

    ld_xor: tile bits XOR-ed into every load address (the first sweep after a
    localized remap reads region alpha of the swapped bits as region 0; the
    bits are tile bits, so every tile still reads only its own positions).

    zero_init: 0 = load the state; 1 = the input is |0...0> with the unit
    amplitude on this device (synthesise tiles, no loads); 2 = the input is
    all zeros on this device.

    sparse = (support, full_out): the run started from |0...0> and only
    amplitudes whose physical bits outside `support` are all 0 can be
    nonzero (support None: every amplitude of this device is 0; see
    program.sparse_start).  Only the tiles whose fixed bits lie inside the
    support are computed ("live" tiles, enumerated compactly); their loads
    of positions outside the support are zero-filled without touching
    memory.  full_out: the next sweep reads the whole state, so every
    position of a dead tile is written with zeros (coalesced streaming
    stores, no loads, no arithmetic); otherwise dead tiles are not touched
    (the next sweep never reads them)."""
    K, D = desc["K"], desc["D"]
    rb = int(desc.get("rb", prog.RB)) if hasattr(desc, "get") else int(desc["rb"])
    NR = 1 << rb
    NT = 1 << (K - rb)
    tin = list(desc["tin"])[:K]
    sw = list(desc["sw"])[:K]
    st_dev = list(desc["st_dev"])[:K]
    st_sw = list(desc["st_sw"])[:K]
    st_flip = int(desc["st_flip"])
    nct = int(desc["nctab"])
    fbits = [b for b in range(D) if b not in tin]
    # chunk bits: fixed per launch (runtime part_val) so a sweep can run in
    # parts that overlap a remap; the tile index enumerates the other bits
    cbits = [b for b in desc.get("cbits", ()) if b in fbits] if hasattr(desc, "get") else []
    fprime = [b for b in fbits if b not in cbits]
    fpos = {b: i for i, b in enumerate(fbits)}
    tb = K - rb  # thread bits
    tinmask = sum(1 << b for b in tin)
    assert not ld_xor & ~tinmask, "load XOR must stay within the tile"
    xr = f" ^ {ld_xor}ull" if ld_xor else ""
    ld_zero = 0  # tile bits whose loaded amplitudes are known zero (zero-filled)
    NTV = "ntiles"  # tiles this launch enumerates
    dead_slabs = []  # (fixed bit set to 1, free bits) covering the dead positions
    if sparse is not None:
        supp, full_out = sparse
        assert not cbits, "sparse sweeps never run in parts"
        if supp is None:
            fprime = []
            NTV = "0ll"
            if full_out:
                dead_slabs = [(None, list(range(D)))]
        else:
            fprime = [b for b in fbits if (supp >> b) & 1]
            NTV = f"{1 << len(fprime)}ll"
            ld_zero = tinmask & ~supp
            if full_out:
                zs = sorted((b for b in fbits if not (supp >> b) & 1), reverse=True)
                for j, z in enumerate(zs):
                    dead_slabs.append((z, [b for b in range(D) if b not in zs[:j + 1]]))

    L = []
    w = L.append
    _pool_begin()
    w('#include "sweep_jit.cuh"')
    _emit_check(w, D)
    w(f"// prefetch={os.environ.get('SVB200_JIT_PREFETCH', 'early')}")
    # sweeps that run beside an overlapped remap leave each SM sub-partition
    # room for the remap's one-warp CTA (48 registers): 2 sweep warps per
    # sub-partition x MAXREG_OVERLAP + 48 must fit in its 16K registers
    if desc.get("cbits") and MAXREG_OVERLAP:
        w(f'extern "C" __global__ void __maxnreg__({MAXREG_OVERLAP})')
    else:
        w(f'extern "C" __global__ void __launch_bounds__({NT}, 1)')
    w(f"{name}(double2* __restrict__ state, const double2* __restrict__ tab, "
      "const svb_cterm* __restrict__ cterms, const int* __restrict__ cofs, double* __restrict__ norm_out, "
      "const u64 part_val, const u64 part_tid, const long long ntiles) {")
    w("  extern __shared__ __align__(16) double2 smem[];")
    w("  __shared__ double red[32];")
    w("  const int t = threadIdx.x;")
    # per-tile slots are double-buffered by tile parity: the next tile's slots
    # are written while slow warps may still read this tile's (no barrier
    # between consecutive tiles)
    w(f"  double2* const ctab_base = smem + {3 << K};")
    # per-thread constants
    w(f"  const u64 ld_t = {_deposit('t', tin[:tb])};")
    w(f"  const u32 lds_t = {_xor_img('t', sw[:tb])};")
    w(f"  const u64 st_t = {_deposit('t', st_dev[:tb])};")
    w(f"  const u32 sts_t = {_xor_img('t', st_sw[:tb])};")
    if ld_zero:
        w(f"  const bool ld_live = (ld_t & {ld_zero}ull) == 0ull;")
    # per-thread phase tables do not depend on the tile: load them once
    for off in sorted({int(op["tab"]) for op in ops if op["kind"] != prog.OP_STAGE and int(op["tab"]) >= 0}):
        w(f"  const double2 tab{off} = __ldg(tab + {off} + t);")
    stages = [op for op in ops if op["kind"] == prog.OP_STAGE]
    stage_info = []
    for si, st in enumerate(stages):
        rm = int(st["rmask"])
        regs = [k for k in range(K) if (rm >> k) & 1]
        flags = int(st["flags"]) if not isinstance(st, dict) else int(st.get("flags", 0))
        if flags & prog.F_TORDER:  # thread-bit order chosen by the planner
            comp = prog.unpack_order(int(st["pval"]), K - len(regs))
        else:
            comp = [k for k in range(K) if not (rm >> k) & 1]
        w(f"  const u32 sb{si} = {_xor_img('t', [sw[k] for k in comp])};")
        w(f"  const u64 db{si} = {_deposit('t', [tin[k] for k in comp])};")
        offs = []
        for v in range(NR):
            o = 0
            for q in range(rb):
                if (v >> q) & 1:
                    o ^= sw[regs[q]]
            offs.append(o)
        stage_info.append((regs, comp, offs))
    # sparse sweeps: positions outside the support are neither loaded nor
    # read back in the first stage (zeros in registers); without a stage the
    # tile is stored straight from shared memory and needs the zero fill
    skip_dead = SKIP_DEAD and bool(ld_zero) and bool(stage_info)
    zk = {k for k in range(K) if (ld_zero >> tin[k]) & 1}
    # tile bits (indices into tin) that may be 1 at a nonzero amplitude: the
    # support inside the tile, grown by the ops that mix a dead bit in
    # (_emit_op zm); all bits of a |0...0> start are dead
    track = ZERO_TRACK and not SPLIT_STAGES and (bool(ld_zero) or bool(zero_init))
    live = set(range(K)) if not track else (set() if zero_init else set(range(K)) - zk)

    def zmask(si):
        return sum(1 << q for q, k in enumerate(stage_info[si][0]) if k not in live)

    def tdead(si):  # thread bits on dead tile bits: such a thread holds zeros only
        return sum(1 << i for i, k in enumerate(stage_info[si][1]) if k not in live)

    def emit_stage_read(si, offs):
        regs, comp, _ = stage_info[si]
        if si != 0 or not skip_dead:
            zm = zmask(si)
            for v in range(NR):
                if v & zm:
                    w(f"    x[{v}] = make_double2(0.0, 0.0);")
                else:
                    w(f"    x[{v}] = tile[sb{si} ^ {offs[v]}u];")
            return
        tmask = sum(1 << i for i, k in enumerate(comp) if k in zk)
        if tmask:
            w(f"    const bool s0_live = (t & {tmask}) == 0;")
        for v in range(NR):
            dead = any((v >> q) & 1 and regs[q] in zk for q in range(rb))
            if dead:
                w(f"    x[{v}] = make_double2(0.0, 0.0);")
            elif tmask:
                w(f"    x[{v}] = s0_live ? tile[sb{si} ^ {offs[v]}u] : make_double2(0.0, 0.0);")
            else:
                w(f"    x[{v}] = tile[sb{si} ^ {offs[v]}u];")

    # direct stores: the last stage's registers go straight to HBM when its
    # lanes cover output bits 0-3 (every warp store writes whole 256-byte
    # runs), skipping the shared-memory round trip of the store path.  Only
    # for sweeps of two or more stages: a one-stage sweep is HBM-bound and
    # its stores, spread over the next tile through shared memory, measured
    # faster (QFT-30 sweep 3: 3.51 vs 3.57 ms; sweep 2, two stages: 0.97 -> 0.75)
    tout = {sw.index(st_sw[i]): st_dev[i] for i in range(K)}
    direct = False
    if DIRECT_STORE and len(stage_info) >= 2 and K - rb >= 5:
        regs_l, comp_l, _ = stage_info[-1]
        direct = {0, 1, 2, 3} <= {tout[k] for k in comp_l[:5]}
    if direct:
        w(f"  const u64 dst_t = {_deposit('t', [tout[k] for k in comp_l])};")
    # norm partial sums: NORM_ACC independent accumulators per sum, so the
    # per-value terms need not form one serial FP64 chain through the tile
    # (ncu, heaviest QV-30 sweep: the single chain's DFMAs hold 9.8% of the
    # not-issued stall samples, but 4 chains measured no faster)
    nacc = max(1, NORM_ACC)
    w("  double " + ", ".join(["nrm = 0.0"] + [f"nrm_a{i} = 0.0" for i in range(1, nacc)]) + ";")
    if bcast is not None and bcast[2] not in (None, 0):
        w("  double " + ", ".join(["nrm2 = 0.0"] + [f"nrm2_a{i} = 0.0" for i in range(1, nacc)]) + ";")
    rot = {"nrm": 0, "nrm2": 0}

    def acc_name(base):
        """Next accumulator of the sum `base` (round robin)."""
        i = rot[base] % nacc
        rot[base] += 1
        return base if i == 0 else f"{base}_a{i}"
    w(f"  long long tile_id = blockIdx.x;")

    def origin(var):
        dep = _deposit(var, fprime) if fprime else "0ull"
        return f"(({dep}) | part_val)" if cbits else dep

    def full_tid(var):  # index over all fixed bits (per-tile slot LUTs)
        if sparse is not None:
            return f"((long long)({_deposit(var, [fpos[b] for b in fprime])}))" if fprime else "0ll"
        if not cbits:
            return var
        return f"((long long)(({_deposit(var, [fpos[b] for b in fprime])}) | part_tid))"

    TILE = 1 << K
    nst = sum(1 for op in ops if int(op["kind"]) == prog.OP_STAGE)
    nslots = max(nst, 1)

    def chunks(n):  # split range(n) into nslots nearly equal consecutive parts
        return [list(range(n * j // nslots, n * (j + 1) // nslots)) for j in range(nslots)]

    # the whole prefetch of tile i+1 goes out at the start of tile i (a full
    # tile of latency slack); the stores of tile i-1 are spread over the stages
    pf_mode = os.environ.get("SVB200_JIT_PREFETCH", "early")
    if pf_mode == "spread":
        pf_chunks = chunks(NR)
    else:
        pf_chunks = [list(range(NR))] + [[] for _ in range(nslots - 1)]
    st_chunks = [[] for _ in range(nslots)] if direct else chunks(NR)

    def prefetch_items(buf, base, items, commit=True):
        for it in items:
            dev = 0
            s = 0
            for q in range(rb):
                if (it >> q) & 1:
                    dev |= 1 << tin[tb + q]
                    s ^= sw[tb + q]
            if dev & ld_zero:  # outside the support: zero, no memory access
                if not skip_dead:
                    w(f"      cp_async16_zero({buf} + (lds_t ^ {s}u), state);")
            elif ld_zero and skip_dead:
                w(f"      if (ld_live) cp_async16({buf} + (lds_t ^ {s}u), state + chk(({base} | ld_t | {dev}ull){xr}));")
            elif ld_zero:
                w(f"      cp_async16_pred({buf} + (lds_t ^ {s}u), state + chk(({base} | ld_t | {dev}ull){xr}), "
                  "ld_live, state);")
            else:
                w(f"      cp_async16({buf} + (lds_t ^ {s}u), state + chk(({base} | ld_t | {dev}ull){xr}));")
        if commit and items:
            w("      cp_async_commit();")

    if bcast is not None:
        bmask, bchains, boff, _ = bcast
        bbits = [b for b in range(D) if (bmask >> b) & 1]
        bcombos = [sum(1 << bbits[i] for i in range(len(bbits)) if (m >> i) & 1) for m in range(1 << len(bbits))]

    def emit_store(val, addr, pred=None, zero=False, ind="        "):
        """One output value: norm terms, then its streaming store(s).  With
        bcast, the copy at combination f is v times f's constants in the
        order the merged sweep would multiply them (bit-identical values)."""
        if bcast is None:
            if not zero:
                a = acc_name("nrm")
                w(f"{ind}{a} = fma({val}.x, {val}.x, fma({val}.y, {val}.y, {a}));")
            if pred is None:
                w(f"{ind}st_stream(state + chk({addr}), {val});")
            else:
                w(f"{ind}if ({pred})")
                w(f"{ind}  st_stream(state + chk({addr}), {val});")
            return
        names = {}
        copies = []
        for f in bcombos:
            ch = bchains.get(f)
            if zero or ch is None:
                copies.append((f, "make_double2(0.0, 0.0)", False))
                continue
            key = tuple(ch)
            if key not in names:
                e = val
                for c in ch:
                    e = _cmul_lit(e, c)
                names[key] = f"cv{len(names)}_"
                w(f"        const double2 {names[key]} = {e};")
            copies.append((f, names[key], True))
        if not zero and (boff is None or boff != 0):  # this sweep's own leaf: every value
            a = acc_name("nrm")
            w(f"        {a} = fma(({val}).x, ({val}).x, fma(({val}).y, ({val}).y, {a}));")
        if pred is not None:
            w(f"        if ({pred}) {{")
        if boff is not None:  # the merged leaf: the values stored (equal copies summed once)
            mult = {}
            for f, cv, live in copies:
                if live:
                    mult[cv] = mult.get(cv, 0) + 1
            for cv, m in mult.items():
                a = acc_name("nrm" if boff == 0 else "nrm2")
                sq = f"fma({cv}.x, {cv}.x, {cv}.y * {cv}.y)"
                w(f"        {a} = fma({_lit_raw(float(m))}, {sq}, {a});" if m > 1 else f"        {a} += {sq};")
        for f, cv, live in copies:
            # the positions' F bits are cleared first: a kept region (st_keep) may set them
            w(f"        st_stream(state + chk((({addr}) & {~bmask & ((1 << 64) - 1)}ull) | {f}ull), {cv});")
        if pred is not None:
            w("        }")

    def store_items(buf, base, items):
        for it in items:
            dev = 0
            s = 0
            for q in range(rb):
                if (it >> q) & 1:
                    dev |= 1 << st_dev[tb + q]
                    s ^= st_sw[tb + q]
            w("      {")
            w(f"        const double2 v = {buf}[sts_t ^ {s}u];")
            pred = None
            if st_keep is not None:
                km, kv = st_keep
                pred = f"((st_t ^ {dev ^ st_flip}ull) & {km}ull) == {kv}ull"
            emit_store("v", f"{base} | ((st_t | {dev}ull) ^ {st_flip}ull)", pred)
            w("      }")

    def slot(j):
        """Issue slice j of the next tile's prefetch and of the previous tile's store."""
        if pf_chunks[j] and not zero_init:
            w("    if (has_next) {")
            prefetch_items("nbuf", "bn", pf_chunks[j])
            w("    }")
        if st_chunks[j]:
            w("    if (iter > 0) {")
            store_items("pbuf", "bp", st_chunks[j])
            w("    }")

    # Three tile buffers rotate: tile i is computed in buffer i % 3 while the
    # prefetch of tile i+1 and the store of tile i-1 are issued in slices
    # between its stages, so loads, stores and FP64 work overlap.
    def emit_ctab(tvar, bvar, dst, per_thread):
        """Per-tile slots of tile `tvar` (origin `bvar`) into `dst`: the
        product of the LUT entries of its index chunks and residual terms."""
        lut_off, nch = int(desc["lut_off"]), int(desc["lut_nch"])
        residual = desc["residual"]
        w(f"    {{ const long long ftid_ = {full_tid(tvar)};")
        w(f"    for (int i = t; i < {nct}; i += {NT}) {{")
        w(f"      const double2* lt = tab + {lut_off} + i * {nch * 256};")
        w("      double2 acc = __ldg(lt + (ftid_ & 255));")
        for c in range(1, nch):
            w(f"      acc = cmul(acc, __ldg(lt + {c * 256} + ((ftid_ >> {8 * c}) & 255)));")
        emit_residual("i", bvar)
        w(f"      {dst}[i] = acc;")
        w("    } }")

    def emit_residual(ivar, bvar):
        residual = desc["residual"]
        if any(residual):
            for s_, terms in enumerate(residual):
                if not terms:
                    continue
                w(f"      if ({ivar} == {s_}) {{")
                for mask, cval in terms:
                    w(f"        if (({bvar} & {int(mask)}ull) == {int(mask)}ull) "
                      f"acc = cmulc(acc, {_lit(cval.real)}, {_lit(cval.imag)});")
                w("      }")

    if nct and nct <= NT and CTAB_AHEAD and not (zero_init and NO_AHEAD_ZERO):  # slots of this CTA's first tile
        w(f"  if (tile_id < {NTV}) {{")
        w(f"    const u64 b0c = {origin('tile_id')};")
        emit_ctab("tile_id", "b0c", "ctab_base", per_thread=False)
        w("  }")
    if not zero_init:
        w(f"  if (tile_id < {NTV}) {{")
        w(f"    const u64 b0 = {origin('tile_id')};")
        prefetch_items("smem", "b0", list(range(NR)))
        w("  }")
    w("  int iter = 0;")
    w(f"  for (; tile_id < {NTV}; ++iter, tile_id += gridDim.x) {{")
    w("    const int r3 = iter % 3;")
    w(f"    double2* const tile = smem + r3 * {TILE};")
    w(f"    double2* const nbuf = smem + (r3 == 2 ? 0 : r3 + 1) * {TILE};")
    w(f"    double2* const pbuf = smem + (r3 == 0 ? 2 : r3 - 1) * {TILE};")
    w(f"    const u64 base = {origin('tile_id')};")
    w(f"    double2* const ctab = ctab_base + (iter & 1) * {max(nct, 1)};")
    w(f"    const bool has_next = tile_id + gridDim.x < {NTV};")
    w("    const long long nx = tile_id + gridDim.x;")
    w(f"    const u64 bn = {origin('nx')};")
    w("    const long long px = tile_id - gridDim.x;")
    w(f"    const u64 bp = {origin('px')};")
    ahead = bool(nct) and nct <= NT and CTAB_AHEAD and not (zero_init and NO_AHEAD_ZERO)
    if nct and not ahead:
        emit_ctab("tile_id", "base", "ctab", per_thread=False)
    w("    cp_async_wait_all();")
    w("    __syncthreads();")
    if ahead:  # this tile's slots were written at the end of the previous tile
        w(f"    double2* const ctab_n = ctab_base + ((iter + 1) & 1) * {nct};")
        lut_off, nch = int(desc["lut_off"]), int(desc["lut_nch"])
        w(f"    double2 lutn[{nch}];")
        w(f"    if (has_next && t < {nct}) {{")
        w(f"      const long long ftn = {full_tid('nx')};")
        w(f"      const double2* lt = tab + {lut_off} + t * {nch * 256};")
        for c in range(nch):
            w(f"      lutn[{c}] = __ldg(lt + {c * 256} + ((ftn >> {8 * c}) & 255));")
        w("    }")
    w(f"    double2 x[{NR}];")

    cur = None  # current stage index
    if nst == 0:
        slot(0)
    pending = []  # ops since the last stage

    def flush(half=None):
        if not track or cur is None or half is not None:
            for o in pending:
                _emit_op(w, o, coef, cur, K, rb, half)
            return
        td = tdead(cur)
        if td and pending:  # ops are linear in the thread's own registers
            w(f"    if ((t & {td}u) == 0u) {{")
        for o in pending:
            woke = _emit_op(w, o, coef, cur, K, rb, None, zmask(cur))
            live.update(stage_info[cur][0][q] for q in range(rb) if (woke >> q) & 1)
        if td and pending:
            w("    }")

    def store_regs(si):
        zm = zmask(si)
        _, _, offs = stage_info[si]
        for v in range(NR):
            val = "make_double2(0.0, 0.0)" if v & zm else f"x[{v}]"
            w(f"    tile[sb{si} ^ {offs[v]}u] = {val};")

    def split_slot(a_stage, b_stage):
        """A register slot whose tile bit stays a register bit across the stage
        and that no pending op pairs on: its two halves go through shared
        memory independently, so one half's FP64 work can overlap the other
        half's stores."""
        if not SPLIT_STAGES:
            return None
        ra, rb_ = stage_info[a_stage][0], stage_info[b_stage][0]
        busy = set()
        for o in pending:
            k = int(o["kind"])
            if k in (prog.OP_H, prog.OP_U1, prog.OP_X):
                busy.add(int(o["a"]))
            elif k == prog.OP_U2:
                busy |= {int(o["a"]), int(o["b"])}
        for q, tbit in enumerate(ra):
            if q not in busy and tbit in rb_:
                return q
        return None

    def warp_local(a_stage, b_stage):
        """Changed lane positions [(lane bit, register slot)] when the stage
        change keeps every warp-level thread bit and each lane that changes
        receives a tile bit from a register (None otherwise)."""
        if not SHUFFLE_STAGES or K - rb < 5:
            return None
        ra, ca = stage_info[a_stage][0], stage_info[a_stage][1]
        cb = stage_info[b_stage][1]
        if ca[5:] != cb[5:]:
            return None
        moves = []
        for p in range(5):
            if ca[p] != cb[p]:
                if cb[p] not in ra:
                    return None
                moves.append(p)
        return moves

    def shuffle_stage(a_stage, b_stage, moves):
        """Butterflies: register slot of tile bit cb[p] <-> lane bit p, then a
        compile-time renaming to the next stage's register slots."""
        slots = list(stage_info[a_stage][0])  # slot -> tile bit, updated per butterfly
        ca, cb = stage_info[a_stage][1], stage_info[b_stage][1]
        for p in moves:
            rs = slots.index(cb[p])
            RS = 1 << rs
            w("    {")
            w(f"      const bool up = (t >> {p}) & 1;")
            for v in range(NR):
                if v & RS:
                    continue
                w(f"      {{ const double2 lo = x[{v}], hi = x[{v | RS}]; const double2 snd = up ? lo : hi; "
                  f"double2 rcv; rcv.x = __shfl_xor_sync(0xffffffffu, snd.x, {1 << p}); "
                  f"rcv.y = __shfl_xor_sync(0xffffffffu, snd.y, {1 << p}); "
                  f"x[{v}] = up ? rcv : lo; x[{v | RS}] = up ? hi : rcv; }}")
            w("    }")
            slots[rs] = ca[p]
        rn = stage_info[b_stage][0]
        src = []
        for vn in range(NR):
            vo = 0
            for qn in range(rb):
                if (vn >> qn) & 1:
                    vo |= 1 << slots.index(rn[qn])
            src.append(vo)
        if src != list(range(NR)):
            w("    {")
            w(f"      const double2 y[{NR}] = {{" + ", ".join(f"x[{v}]" for v in src) + "};")
            for v in range(NR):
                w(f"      x[{v}] = y[{v}];")
            w("    }")

    for op in ops:
        kind = int(op["kind"])
        if kind == prog.OP_STAGE:
            nxt = 0 if cur is None else cur + 1
            moves = warp_local(cur, nxt) if cur is not None else None
            if moves is not None:
                flush()
                pending = []
                shuffle_stage(cur, nxt, moves)
                cur = nxt
                slot(nxt)
                continue
            if cur is not None:
                _, _, offs = stage_info[cur]
                q = split_slot(cur, nxt)
                halves = [None] if q is None else [(q, 0), (q, 1)]
                for hf in halves:
                    flush(hf)
                    if hf is None:
                        store_regs(cur)
                        continue
                    for v in range(NR):
                        if ((v >> q) & 1) == hf[1]:
                            w(f"    tile[sb{cur} ^ {offs[v]}u] = x[{v}];")
                w("    __syncwarp();" if _warp_local_change(stage_info, cur, nxt, NT) else "    __syncthreads();")
            else:
                flush()
            pending = []
            _, _, offs = stage_info[nxt]
            if nxt == 0 and zero_init:
                # |0...0>: every amplitude is zero except index 0 of the device
                for v in range(NR):
                    w(f"    x[{v}] = make_double2(0.0, 0.0);")
                if zero_init == 1:
                    w("    if (base == 0ull && t == 0) x[0] = make_double2(1.0, 0.0);")
            else:
                emit_stage_read(nxt, offs)
            cur = nxt
            slot(nxt)
            continue
        pending.append(op)
    flush()
    pending = []

    if cur is not None and direct:
        zm = zmask(cur)
        for v in range(NR):
            dev = sum(1 << tout[regs_l[q]] for q in range(rb) if (v >> q) & 1)
            pred = None
            if st_keep is not None:
                km, kv = st_keep
                pred = f"((dst_t ^ {dev ^ st_flip}ull) & {km}ull) == {kv}ull"
            w("    {")
            emit_store("make_double2(0.0, 0.0)" if v & zm else f"x[{v}]",
                       f"base | ((dst_t | {dev}ull) ^ {st_flip}ull)", pred, zero=bool(v & zm), ind="      ")
            w("    }")
    elif cur is not None:
        store_regs(cur)
    if ahead:  # the next tile's slots, from loads issued at the start of this one
        nch = int(desc["lut_nch"])
        w(f"    if (has_next && t < {nct}) {{")
        w("      double2 acc = lutn[0];")
        for c in range(1, nch):
            w(f"      acc = cmul(acc, lutn[{c}]);")
        emit_residual("t", "bn")
        w("      ctab_n[t] = acc;")
        w("    }")
    w("  }")
    # the last tile of this CTA is still in shared memory
    w("  __syncthreads();")
    w(f"  if ({'false' if direct else 'iter > 0'}) {{")
    w(f"    double2* const pbuf = smem + ((iter - 1) % 3) * {TILE};")
    w("    const long long px = tile_id - gridDim.x;")
    w(f"    const u64 bp = {origin('px')};")
    store_items("pbuf", "bp", list(range(NR)))
    w("  }")
    w("  cp_async_wait_all();")
    for z, free in dead_slabs:  # dead positions of a sparse sweep: zeros
        n = 1 << len(free)
        one = f" | {1 << z}ull" if z is not None else ""
        w("  {")
        w(f"    const long long gs = (long long)gridDim.x * {NT};")
        w(f"    for (long long c = (long long)blockIdx.x * {NT} + t; c < {n}ll; c += gs)")
        w(f"      st_stream(state + chk(({_deposit('c', free)}){one}), make_double2(0.0, 0.0));")
        w("  }")
    w("  if (norm_out != nullptr) {")
    full = "0xffffffffu" if NT >= 32 else f"{(1 << NT) - 1}u"
    two = bcast is not None and bcast[2] not in (None, 0)
    for acc, dst, mult in [("nrm", "norm_out", 1)] + ([("nrm2", f"norm_out + {bcast[2]}", 1)] if two else []):
        if nacc == 4:
            w(f"    {acc} = ({acc} + {acc}_a1) + ({acc}_a2 + {acc}_a3);")
        elif nacc > 1:
            w(f"    {acc} = " + " + ".join([acc] + [f"{acc}_a{i}" for i in range(1, nacc)]) + ";")
        for o in (16, 8, 4, 2, 1):
            if o < NT:
                w(f"    {acc} += __shfl_xor_sync({full}, {acc}, {o});")
        w(f"    if ((t & 31) == 0) red[t >> 5] = {acc};")
        w("    __syncthreads();")
        w("    if (t == 0) {")
        w("      double s = 0.0;")
        w(f"      for (int i = 0; i < {(NT + 31) // 32}; ++i) s += red[i];")
        w(f"      atomicAdd({dst}, {_lit_raw(float(mult))} * s);" if mult != 1 else f"      atomicAdd({dst}, s);")
        w("    }")
        if two and acc == "nrm":  # red[] is reused for the second sum
            w("    __syncthreads();")
    w("  }")
    w("}")
    return "\n".join(_pool_end(L)) + "\n"


GROUP_OFFSET = os.environ.get("SVB200_JIT_GROUP_OFFSET", "1") not in ("0", "false", "no")
GROUPS_ONLY = int(os.environ["SVB200_JIT_GROUPS_ONLY"]) if os.environ.get("SVB200_JIT_GROUPS_ONLY") else None
SKIP_DEAD = os.environ.get("SVB200_JIT_SKIP_DEAD", "1") not in ("0", "false", "no")
# norm accumulators per thread (kernel_source); 4 measured equal to 1 on QV-30 and QFT-30
# (655-657 ms, 3.09 ms either way: the chain's stalls are hidden), so the default keeps one
NORM_ACC = int(os.environ.get("SVB200_JIT_NORM_ACC", "1"))
# the last stage stores straight from registers when that coalesces (kernel_source)
DIRECT_STORE = os.environ.get("SVB200_JIT_DIRECT_STORE", "1") not in ("0", "false", "no")
# sparse sweeps: known-zero registers drop out of the arithmetic (kernel_source)
ZERO_TRACK = os.environ.get("SVB200_JIT_ZERO_TRACK", "1") not in ("0", "false", "no")
# sweeps whose FP64 work per amplitude reaches this many DFMA (a fused 4x4 is
# 16) run two tile groups per CTA (kernel_source_2g)
GROUPS_MIN_DFMA = float(os.environ.get("SVB200_JIT_GROUPS_MIN_DFMA", "48"))


def dfma_per_amp(ops, rb: int) -> float:
    """FP64 FMAs per amplitude of a sweep's dense gates: a 4x4 on register
    pairs 16, a 2x2 8 (the tile-group choice; phase-only sweeps stay in one
    group, measured faster on the QFT; the roofline counts SASS instead)."""
    n = 0.0
    for op in ops:
        k = int(op["kind"])
        if k == prog.OP_U2:
            n += 16
        elif k == prog.OP_U1:
            n += 8
    return n


def kernel_source_2g(name: str, desc: dict, ops: list, coef: list, zero_init: int = 0,
                     sparse: tuple | None = None) -> str:
    """Straight-line kernel for one FP64-heavy sweep with two tile groups.

    A one-group CTA cannot overlap a register<->shared-memory stage with
    FP64 work: all its warps meet at the stage barrier (round-1 ncu: FP64
    pipe 67%, the heaviest QV sweep's time = FP64 time + stage time).  Here
    the CTA has two groups of 2^(K-rb) threads working on alternate tiles
    of the CTA's sequence (tile k -> group k % 2, buffer k % 3), each with
    its own named barrier, so one group's stages and stores run while the
    other computes.  Loads are cp.async into the buffer of tile k+3, issued
    by the group that just stored tile k from that buffer and tracked by an
    mbarrier per tile index mod 6 (cp.async.mbarrier.arrive): the consumer
    of tile k waits on barrier k mod 6 with parity (k / 6) & 1.  Six
    barriers, not one per buffer: a parity wait cannot tell phase j from
    phase j - 2, and with one barrier per buffer a consumer could reach
    tile k + 3 while the loads of tile k were still in flight and take
    them as complete (found on light QFT sweeps, tools/kernel_ab.py);
    barrier k mod 6 was last waited on by the same group for tile k - 6,
    so its previous phase is always complete.  Registers: 512
    threads leave 128 per thread."""
    K, D = desc["K"], desc["D"]
    rb = int(desc["rb"])
    NR = 1 << rb
    NT = 1 << (K - rb)
    tb = K - rb
    tin = list(desc["tin"])[:K]
    sw = list(desc["sw"])[:K]
    st_dev = list(desc["st_dev"])[:K]
    st_sw = list(desc["st_sw"])[:K]
    st_flip = int(desc["st_flip"])
    nct = int(desc["nctab"])
    assert not desc.get("cbits"), "part launches keep the one-group kernel"
    fbits = [b for b in range(D) if b not in tin]
    fpos = {b: i for i, b in enumerate(fbits)}
    fprime = list(fbits)
    tinmask = sum(1 << b for b in tin)
    ld_zero = 0
    NTV = "ntiles"
    dead_slabs = []
    if sparse is not None:
        supp, full_out = sparse
        if supp is None:
            fprime = []
            NTV = "0ll"
            if full_out:
                dead_slabs = [(None, list(range(D)))]
        else:
            fprime = [b for b in fbits if (supp >> b) & 1]
            NTV = f"{1 << len(fprime)}ll"
            ld_zero = tinmask & ~supp
            if full_out:
                zs = sorted((b for b in fbits if not (supp >> b) & 1), reverse=True)
                for j, z in enumerate(zs):
                    dead_slabs.append((z, [b for b in range(D) if b not in zs[:j + 1]]))

    def origin(var):
        return _deposit(var, fprime) if fprime else "0ull"

    def full_tid(var):
        if sparse is not None:
            return f"((long long)({_deposit(var, [fpos[b] for b in fprime])}))" if fprime else "0ll"
        return var

    L = []
    w = L.append
    _pool_begin()
    w('#include "sweep_jit.cuh"')
    _emit_check(w, D)
    w("// two tile groups")
    w(f'extern "C" __global__ void __launch_bounds__({2 * NT}, 1)')
    w(f"{name}(double2* __restrict__ state, const double2* __restrict__ tab, "
      "const svb_cterm* __restrict__ cterms, const int* __restrict__ cofs, double* __restrict__ norm_out, "
      "const u64 part_val, const u64 part_tid, const long long ntiles) {")
    w("  extern __shared__ __align__(16) double2 smem[];")
    w("  __shared__ double red[32];")
    w("  __shared__ __align__(8) unsigned long long mbar[6];")
    w(f"  const int grp = threadIdx.x >> {tb};")
    w(f"  const int t = threadIdx.x & {NT - 1};")
    w("  const u32 bar_id = 1u + (u32)grp;")
    w(f"  double2* const ctab = smem + {3 << K} + grp * {max(nct, 1)};")
    w(f"  const u64 ld_t = {_deposit('t', tin[:tb])};")
    w(f"  const u32 lds_t = {_xor_img('t', sw[:tb])};")
    w(f"  const u64 st_t = {_deposit('t', st_dev[:tb])};")
    w(f"  const u32 sts_t = {_xor_img('t', st_sw[:tb])};")
    if ld_zero:
        w(f"  const bool ld_live = (ld_t & {ld_zero}ull) == 0ull;")
    for off in sorted({int(op["tab"]) for op in ops if op["kind"] != prog.OP_STAGE and int(op["tab"]) >= 0}):
        w(f"  const double2 tab{off} = __ldg(tab + {off} + t);")
    stages = [op for op in ops if op["kind"] == prog.OP_STAGE]
    stage_info = []
    for si, st in enumerate(stages):
        rm = int(st["rmask"])
        regs = [k for k in range(K) if (rm >> k) & 1]
        flags = int(st["flags"]) if not isinstance(st, dict) else int(st.get("flags", 0))
        if flags & prog.F_TORDER:
            comp = prog.unpack_order(int(st["pval"]), K - len(regs))
        else:
            comp = [k for k in range(K) if not (rm >> k) & 1]
        w(f"  const u32 sb{si} = {_xor_img('t', [sw[k] for k in comp])};")
        w(f"  const u64 db{si} = {_deposit('t', [tin[k] for k in comp])};")
        offs = []
        for v in range(NR):
            o = 0
            for q in range(rb):
                if (v >> q) & 1:
                    o ^= sw[regs[q]]
            offs.append(o)
        stage_info.append((regs, comp, offs))
    TILE = 1 << K
    skip_dead = SKIP_DEAD and bool(ld_zero) and bool(stage_info)
    zk = {k for k in range(K) if (ld_zero >> tin[k]) & 1}

    def emit_stage_read(si, offs):
        regs, comp, _ = stage_info[si]
        if si != 0 or not skip_dead:
            for v in range(NR):
                w(f"    x[{v}] = tile[sb{si} ^ {offs[v]}u];")
            return
        tmask = sum(1 << i for i, k in enumerate(comp) if k in zk)
        if tmask:
            w(f"    const bool s0_live = (t & {tmask}) == 0;")
        for v in range(NR):
            dead = any((v >> q) & 1 and regs[q] in zk for q in range(rb))
            if dead:
                w(f"    x[{v}] = make_double2(0.0, 0.0);")
            elif tmask:
                w(f"    x[{v}] = s0_live ? tile[sb{si} ^ {offs[v]}u] : make_double2(0.0, 0.0);")
            else:
                w(f"    x[{v}] = tile[sb{si} ^ {offs[v]}u];")

    def prefetch_items(buf, base):
        for it in range(NR):
            dev = 0
            s_ = 0
            for q in range(rb):
                if (it >> q) & 1:
                    dev |= 1 << tin[tb + q]
                    s_ ^= sw[tb + q]
            if dev & ld_zero:  # outside the support: zero, no memory access
                if not skip_dead:
                    w(f"      cp_async16_zero({buf} + (lds_t ^ {s_}u), state);")
            elif ld_zero and skip_dead:
                w(f"      if (ld_live) cp_async16({buf} + (lds_t ^ {s_}u), state + chk({base} | ld_t | {dev}ull));")
            elif ld_zero:
                w(f"      cp_async16_pred({buf} + (lds_t ^ {s_}u), state + chk({base} | ld_t | {dev}ull), "
                  "ld_live, state);")
            else:
                w(f"      cp_async16({buf} + (lds_t ^ {s_}u), state + chk({base} | ld_t | {dev}ull));")

    w("  if (threadIdx.x == 0) {")
    w("    for (int b = 0; b < 6; ++b) mbar_init(&mbar[b], " + str(NT) + "u);")
    w("    mbar_init_fence();")
    w("  }")
    w("  __syncthreads();")
    w("  double nrm = 0.0;")
    if not zero_init:
        # tiles 0 and 2 by group 0, tile 1 by group 1 (buffer = tile % 3)
        w("  for (int k = grp; k < 3; k += 2) {")
        w("    const long long pt = blockIdx.x + (long long)k * gridDim.x;")
        w(f"    if (pt < {NTV}) {{")
        w(f"      const u64 bq = {origin('pt')};")
        prefetch_items(f"(smem + k * {TILE})", "bq")
        w("    }")
        w("    cp_async_mbar_arrive(&mbar[k]);")
        w("  }")
    # start the groups half a tile apart: group 1 waits until group 0 is in
    # the middle of its first tile, so one group's stages and stores fall in
    # the other's FP64 phase (started together they stay in lockstep)
    nst = len(stage_info)
    mid = nst // 2 if (nst >= 2 and GROUP_OFFSET) else None
    if mid is not None:
        w("  bool offset_pending = grp == 0;")
        w(f"  if (grp == 1) bar_group(3u, {2 * NT}u);")
    w("  for (int k = grp;; k += 2) {")
    w("    const long long tile_id = blockIdx.x + (long long)k * gridDim.x;")
    w(f"    if (tile_id >= {NTV}) break;")
    w("    const int b = k % 3;")
    w(f"    double2* const tile = smem + b * {TILE};")
    w(f"    const u64 base = {origin('tile_id')};")
    if nct:
        lut_off, nch = int(desc["lut_off"]), int(desc["lut_nch"])
        residual = desc["residual"]
        w(f"    {{ const long long ftid_ = {full_tid('tile_id')};")
        w(f"    for (int i = t; i < {nct}; i += {NT}) {{")
        w(f"      const double2* lt = tab + {lut_off} + i * {nch * 256};")
        w("      double2 acc = __ldg(lt + (ftid_ & 255));")
        for c in range(1, nch):
            w(f"      acc = cmul(acc, __ldg(lt + {c * 256} + ((ftid_ >> {8 * c}) & 255)));")
        if any(residual):
            for s_, terms in enumerate(residual):
                if not terms:
                    continue
                w(f"      if (i == {s_}) {{")
                for mask, cval in terms:
                    w(f"        if ((base & {int(mask)}ull) == {int(mask)}ull) "
                      f"acc = cmulc(acc, {_lit(cval.real)}, {_lit(cval.imag)});")
                w("      }")
        w("      ctab[i] = acc;")
        w("    } }")
    if not zero_init:
        w("    mbar_wait_parity(&mbar[k % 6], (u32)((k / 6) & 1));")
    w(f"    bar_group(bar_id, {NT}u);")
    w(f"    double2 x[{NR}];")
    cur = None
    pending = []
    for op in ops:
        kind = int(op["kind"])
        if kind == prog.OP_STAGE:
            nxt = 0 if cur is None else cur + 1
            for o in pending:
                _emit_op(w, o, coef, cur, K, rb)
            pending = []
            if cur is not None:
                _, _, offs = stage_info[cur]
                for v in range(NR):
                    w(f"    tile[sb{cur} ^ {offs[v]}u] = x[{v}];")
                if _warp_local_change(stage_info, cur, nxt, NT):
                    w("    __syncwarp();")
                else:
                    w(f"    bar_group(bar_id, {NT}u);")
            _, _, offs = stage_info[nxt]
            if nxt == 0 and zero_init:
                for v in range(NR):
                    w(f"    x[{v}] = make_double2(0.0, 0.0);")
                if zero_init == 1:
                    w("    if (base == 0ull && t == 0) x[0] = make_double2(1.0, 0.0);")
            else:
                emit_stage_read(nxt, offs)
            if nxt == mid:
                w(f"    if (offset_pending) {{ bar_group(3u, {2 * NT}u); offset_pending = false; }}")
            cur = nxt
            continue
        pending.append(op)
    for o in pending:
        _emit_op(w, o, coef, cur, K, rb)
    if cur is not None:
        _, _, offs = stage_info[cur]
        for v in range(NR):
            w(f"    tile[sb{cur} ^ {offs[v]}u] = x[{v}];")
    w(f"    bar_group(bar_id, {NT}u);")
    for it in range(NR):  # store this tile, then the buffer takes tile k+3
        dev = 0
        s_ = 0
        for q in range(rb):
            if (it >> q) & 1:
                dev |= 1 << st_dev[tb + q]
                s_ ^= st_sw[tb + q]
        w("    {")
        w(f"      const double2 v = tile[sts_t ^ {s_}u];")
        w("      nrm = fma(v.x, v.x, fma(v.y, v.y, nrm));")
        w(f"      st_stream(state + chk(base | ((st_t | {dev}ull) ^ {st_flip}ull)), v);")
        w("    }")
    if not zero_init:
        w(f"    bar_group(bar_id, {NT}u);")
        w("    {")
        w("      const long long nk = tile_id + 3ll * gridDim.x;")
        w(f"      if (nk < {NTV}) {{")
        w(f"        const u64 bn = {origin('nk')};")
        prefetch_items("tile", "bn")
        w("      }")
        w("      cp_async_mbar_arrive(&mbar[(k + 3) % 6]);")
        w("    }")
    w("  }")
    if mid is not None:  # group 0 had no tile: release group 1
        w(f"  if (offset_pending) bar_group(3u, {2 * NT}u);")
    w("  cp_async_wait_all();")
    for z, free in dead_slabs:
        n = 1 << len(free)
        one = f" | {1 << z}ull" if z is not None else ""
        w("  {")
        w(f"    const long long gs = (long long)gridDim.x * {2 * NT};")
        w(f"    for (long long c = (long long)blockIdx.x * {2 * NT} + threadIdx.x; c < {n}ll; c += gs)")
        w(f"      st_stream(state + chk(({_deposit('c', free)}){one}), make_double2(0.0, 0.0));")
        w("  }")
    w("  if (norm_out != nullptr) {")
    for o in (16, 8, 4, 2, 1):
        w(f"    nrm += __shfl_xor_sync(0xffffffffu, nrm, {o});")
    w("    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;")
    w("    __syncthreads();")
    w("    if (threadIdx.x == 0) {")
    w("      double s = 0.0;")
    w(f"      for (int i = 0; i < {2 * NT // 32}; ++i) s += red[i];")
    w("      atomicAdd(norm_out, s);")
    w("    }")
    w("  }")
    w("}")
    return "\n".join(_pool_end(L)) + "\n"


# SVB200_JIT_CHECK=1: every global state index of a generated kernel is
# bounds-checked (trap) against the device's 2^D amplitudes -- the self-check
# mode that replaces compute-sanitizer on pools where it is unavailable
CHECK = os.environ.get("SVB200_JIT_CHECK", "0") not in ("0", "false", "no")


def _emit_check(w, D: int) -> None:
    if CHECK:
        w(f"SVB_F u64 chk(u64 i) {{ if (i >= {1 << D}ull) __trap(); return i; }}")
    else:
        w("#define chk(i) (i)")


def _phase_base(w, op, coef_c0: complex, K: int, rb: int) -> None:
    """Emit `p` = const * per-tile slot * per-thread table * per-thread-bit slots.

    A unit constant is not multiplied (x * 1 is not folded by the compiler
    under IEEE rules)."""
    factors = []
    if int(op["ctab"]) >= 0:
        factors.append(f"ctab[{int(op['ctab'])}]")
    if int(op["tab"]) >= 0:
        factors.append(f"tab{int(op['tab'])}")
    c0 = complex(coef_c0)
    if not factors:
        w(f"      double2 p = make_double2({_lit(c0.real)}, {_lit(c0.imag)});")
    else:
        w(f"      double2 p = {factors[0]};")
        for f in factors[1:]:
            w(f"      p = cmul(p, {f});")
        if c0 != 1:
            w(f"      p = {_cmul_lit('p', c0)};")
    if int(op["tf"]) >= 0:
        for i in range(K - rb):
            w(f"      if ((t >> {i}) & 1) p = cmul(p, ctab[{int(op['tf']) + i}]);")


def _emit_op(w, op, coef, stage, K, rb, half=None, zm: int = 0) -> int:
    """Emit one op; `half` = (register slot, value) restricts it to the
    amplitudes whose slot bit has that value (ops that do not pair across
    that slot split exactly into two halves).

    zm: register slots whose tile bit is still dead (register v holds an
    exact zero whenever v & zm; kernel_source tracks this from the sparse
    support).  Terms on such registers are dropped: a butterfly with a zero
    partner becomes a copy, a phase on a zero amplitude is skipped.  Every
    dropped term is an exact zero added or multiplied, so the results equal
    the full computation's (up to the sign of zero).  Returns the slots the
    op makes live."""
    NR = 1 << rb
    kind = int(op["kind"])

    def skip(v):
        return half is not None and ((v >> half[0]) & 1) != half[1]

    def z(v):
        return bool(v & zm)

    a = int(op["a"])
    A = 1 << a
    cm, cv = int(op["rmask"]), int(op["b"])
    cf = int(op["coef"])
    pmask, pval = int(op["pmask"]), int(op["pval"])
    woke = 0
    w("    {")
    if pmask:
        w(f"    if (((base | db{stage}) & {pmask}ull) == {pval}ull) {{")
    if kind in (prog.OP_H, prog.OP_U1, prog.OP_PH):
        has_phase = kind == prog.OP_PH or (int(op["flags"]) & prog.F_PHASE)
        fused = False
        if has_phase:
            ph = cf if kind == prog.OP_PH else cf + 4
            _phase_base(w, op, coef[ph], K, rb)
            nt = (int(op["flags"]) >> prog.F_PREG_SHIFT) & 0xF
            fused = kind == prog.OP_H and cm == 0
            _emit_dfs(w, a, nt, [coef[ph + 1 + s] for s in range(rb)], fused, rb, half, zm)
        if kind == prog.OP_H and not fused:
            for v in range(NR):
                if (v & A) or (v & cm) != cv or skip(v):
                    continue
                z0, z1 = z(v), z(v | A)
                if z0 and z1:
                    continue
                if z1:
                    w(f"      x[{v | A}] = x[{v}];")
                elif z0:
                    w(f"      x[{v}] = x[{v | A}]; x[{v | A}] = make_double2(-x[{v}].x, -x[{v}].y);")
                else:
                    w(f"      {{ const double2 x0 = x[{v}], x1 = x[{v | A}]; "
                      f"x[{v}] = cadd(x0, x1); x[{v | A}] = csub(x0, x1); }}")
        elif kind == prog.OP_U1:
            m00, m01, m10, m11 = coef[cf:cf + 4]
            for v in range(NR):
                if (v & A) or (v & cm) != cv or skip(v):
                    continue
                z0, z1 = z(v), z(v | A)
                if z0 and z1:
                    continue
                t0 = [] if z0 else [(m00, "x0")]
                t1 = [] if z0 else [(m10, "x0")]
                if not z1:
                    t0.append((m01, "x1"))
                    t1.append((m11, "x1"))
                w(f"      {{ const double2 x0 = x[{v}], x1 = x[{v | A}]; "
                  f"x[{v}] = {_lincomb(t0)}; x[{v | A}] = {_lincomb(t1)}; }}")
        if kind in (prog.OP_H, prog.OP_U1):
            woke |= A
    elif kind == prog.OP_X:
        for v in range(NR):
            if (v & A) or (v & cm) != cv or skip(v):
                continue
            if z(v) and z(v | A):
                continue
            w(f"      {{ const double2 tmp = x[{v}]; x[{v}] = x[{v | A}]; x[{v | A}] = tmp; }}")
        woke |= A  # the zero half moves to bit value 0: no longer "bit set -> zero"
    elif kind == prog.OP_U2:
        b = int(op["b"])
        B = 1 << b
        M = np.asarray(coef[cf:cf + 16]).reshape(4, 4)
        D = _column_phases(M) if FACTOR_U2 else None
        if D is not None:  # M = R diag(D), R real/imaginary: 4 + 8 instead of 16 FP64 per amplitude
            M = M / D[None, :]
            M = np.where(np.abs(M.imag) <= 1e-15 * np.abs(M), M.real + 0j,
                         np.where(np.abs(M.real) <= 1e-15 * np.abs(M), 1j * M.imag, M))
        for v in range(NR):
            if (v & A) or (v & B) or skip(v):
                continue
            idx = [v, v | B, v | A, v | A | B]
            live = [c for c in range(4) if not z(idx[c])]
            if not live:
                continue
            w("      {")
            if D is None:
                w("        const double2 " + ", ".join(f"a{c} = x[{idx[c]}]" for c in live) + ";")
            else:
                w("        const double2 " + ", ".join(f"a{c} = {_cmul_lit(f'x[{idx[c]}]', D[c])}" for c in live)
                  + ";")
            for r in range(4):
                w(f"        x[{idx[r]}] = {_lincomb([(M[r, c], f'a{c}') for c in live])};")
            w("      }")
        woke |= A | B
    elif kind == prog.OP_PHALL:
        _phase_base(w, op, coef[cf], K, rb)
        for v in range(NR):
            if not skip(v) and not z(v):
                w(f"      x[{v}] = cmul(x[{v}], p);")
    elif kind == prog.OP_SCALE:
        for v in range(NR):
            if not skip(v) and not z(v):
                w(f"      x[{v}] = {_cmul_lit(f'x[{v}]', coef[cf])};")
    if pmask:
        w("    }")
    w("    }")
    return woke & zm


# a 4x4 whose columns are each a phase times a real/imaginary vector (QAOA:
# rx (x) rx after a ZZ phase) runs as a diagonal then a real/imaginary 4x4
FACTOR_U2 = os.environ.get("SVB200_JIT_FACTOR_U2", "1") not in ("0", "false", "no")


def _column_phases(M: np.ndarray):
    """D with M = R diag(D), every entry of R real or imaginary, when M
    itself is not (else None)."""
    def ri(z):
        return z.real == 0 or z.imag == 0

    if all(ri(z) for z in M.ravel()):
        return None
    D = np.ones(4, dtype=np.complex128)
    for c in range(4):
        col = M[:, c]
        nz = [z for z in col if z != 0]
        if not nz:
            continue
        ph = nz[0] / abs(nz[0])
        q = col / ph
        # entries within rounding of the real or imaginary axis count; the
        # factored product equals M to ~1 ulp (checked by the parity tests)
        if not all(abs(z.imag) <= 1e-15 * abs(z) or abs(z.real) <= 1e-15 * abs(z) for z in q):
            return None
        D[c] = ph
    return D


def _emit_dfs(w, a: int, nt: int, c: list, fused_h: bool, rb: int, half=None, zm: int = 0) -> None:
    """Depth-first product over register slots != a; leaves are amplitudes with bit a set
    (zm: see _emit_op; unused partial products are dead code)."""
    counter = [0]

    def rec(s, v, pv):
        if s == rb:
            if half is not None and ((v >> half[0]) & 1) != half[1]:
                return  # the other half (unused partial products are dead code)
            u = v ^ (1 << a)
            if fused_h:
                if v & zm and u & zm:
                    return
                if v & zm:  # x1 = 0: both outputs are x0
                    w(f"      x[{v}] = x[{u}];")
                elif u & zm:  # x0 = 0
                    w(f"      x[{u}] = cmul(x[{v}], {pv}); x[{v}] = make_double2(-x[{u}].x, -x[{u}].y);")
                else:
                    w(f"      {{ const double2 x1 = cmul(x[{v}], {pv}); const double2 x0 = x[{u}]; "
                      f"x[{u}] = cadd(x0, x1); x[{v}] = csub(x0, x1); }}")
            elif not v & zm:
                w(f"      x[{v}] = cmul(x[{v}], {pv});")
            return
        if s == a:
            rec(s + 1, v, pv)
            return
        rec(s + 1, v, pv)
        if (nt >> s) & 1:
            counter[0] += 1
            q = f"q{counter[0]}"
            w(f"      const double2 {q} = {_cmul_lit(pv, c[s])};")
            rec(s + 1, v | (1 << s), q)
        else:
            rec(s + 1, v | (1 << s), pv)

    rec(0, 1 << a, "p")


# ---------------------------------------------------------------------------
# compile / load / launch
# ---------------------------------------------------------------------------

_mem_cache: dict = {}  # source hash -> cubin bytes
_LAST_ZERO_INIT: dict = {}  # descriptors the last build_kernels synthesised from |0>
_LAST_GROUPS: dict = {}  # descriptors the last build_kernels rendered with two tile groups
_kernels: dict = {}  # (source hash, device) -> kernel handle


_HEADER_KEY = None


def _header_key() -> str:
    """Content of the headers the generated source includes (part of the cache key)."""
    global _HEADER_KEY
    if _HEADER_KEY is None:
        _HEADER_KEY = "".join((CSRC / f).read_text() for f in ("sweep_jit.cuh",))
    return _HEADER_KEY


def _key(src: str) -> str:
    return hashlib.sha256((src + "\0" + " ".join(NVRTC_OPTS) + "\0" + _header_key()).encode()).hexdigest()


def _cached(h: str) -> bytes | None:
    hit = _mem_cache.get(h)
    if hit is not None:
        return hit
    path = CACHE_DIR / f"{h}.cubin"
    try:
        data = path.read_bytes()
    except OSError:
        return None
    _mem_cache[h] = data
    return data


LOCK_STALE_S = 120.0


def _compile(src: str, name: str) -> bytes:
    """NVRTC-compile one kernel, or take it from the memory / disk cache.

    Processes of one node share the disk cache: a kernel another process
    is compiling (its lock file exists) is waited for instead of compiled
    twice, so ranks with identical sweeps split the compile work."""
    h = _key(src)
    hit = _cached(h)
    if hit is not None:
        return hit
    lock = CACHE_DIR / f"{h}.lock"
    try:
        CACHE_DIR.mkdir(parents=True, exist_ok=True)
        fd = os.open(lock, os.O_CREAT | os.O_EXCL | os.O_WRONLY)
        os.close(fd)
        owned = True
    except FileExistsError:
        owned = False
    except OSError:
        owned = True  # no writable cache: compile here
    if not owned:
        import time

        while True:
            hit = _cached(h)
            if hit is not None:
                return hit
            try:
                age = time.time() - lock.stat().st_mtime
            except OSError:
                age = None  # the owner finished (or failed): compile here
            if age is None or age > LOCK_STALE_S:
                break
            time.sleep(0.005)
    try:
        return _nvrtc(src, name, h)
    finally:
        if owned:
            try:
                lock.unlink()
            except OSError:
                pass


def _nvrtc(src: str, name: str, h: str) -> bytes:
    path = CACHE_DIR / f"{h}.cubin"
    lib = _native.load()
    opts = (ctypes.c_char_p * len(NVRTC_OPTS))(*[o.encode() for o in NVRTC_OPTS])
    image = ctypes.c_void_p()
    size = ctypes.c_size_t()
    log = ctypes.create_string_buffer(1 << 16)
    rc = 1
    for attempt in range(2):  # a failure with an empty log (resource exhaustion) is retried once
        rc = lib.svb_jit_compile(src.encode(), name.encode(), len(NVRTC_OPTS), opts, ctypes.byref(image),
                                 ctypes.byref(size), log, len(log))
        if rc == 0 or log.value.strip():
            break
    if rc != 0:
        err = lib.svb_last_error().decode(errors="replace")
        raise _native.NativeError(f"NVRTC failed for {name} ({err}): {log.value.decode(errors='replace')[:4000]}")
    data = ctypes.string_at(image, size.value)
    lib.svb_jit_free(image)
    try:
        CACHE_DIR.mkdir(parents=True, exist_ok=True)
        tmp = path.with_suffix(f".tmp{os.getpid()}")
        tmp.write_bytes(data)
        os.replace(tmp, path)
    except OSError:
        pass
    _mem_cache[h] = data
    return data


def build_kernels(buf: prog.ProgramBuffers, prefix: str = "svb_jit", threads: int | None = None,
                  zero_init: dict | None = None, sparse: dict | None = None, lazy: bool = False,
                  ld_xor: dict | None = None, st_keep: dict | None = None, bcast: dict | None = None,
                  skip=()):
    """Generate + compile one kernel per sweep descriptor; returns (names, cubins).

    bcast: descriptor -> broadcast store (executor._broadcast_merges); skip:
    descriptors merged into the sweep before them (no kernel, name None).

    zero_init maps descriptor index -> 1/2 for sweeps whose input is known to
    be |0...0> (see kernel_source); _LAST_ZERO_INIT records which were used.
    sparse maps descriptor index -> (support, full_out) from
    program.sparse_start (a run from |0...0>); it implies zero_init for the
    sweeps that start from the unit vector or from zeros."""
    srcs, names = [], []
    zero_init = dict(zero_init or {})
    sparse = dict(sparse or {})
    for i, (supp, _) in sparse.items():
        if supp is None or supp == 0:
            zero_init[i] = 2 if supp is None else 1
    used = {}
    groups = {}
    bcast = dict(bcast or {})
    for i, d in enumerate(buf.descs):
        if i in skip:
            names.append(None)
            continue
        ops = buf.ops[d["op_begin"]: d["op_begin"] + d["op_count"]]
        zi = zero_init.get(i, 0)
        if zi and not (zi == 2 and i in sparse) and not any(int(o["kind"]) == prog.OP_STAGE for o in ops):
            raise ValueError(f"sweep {i} cannot synthesise |0...0> (no register stage)")
        if zi:
            used[i] = zi
        two = (GROUPS and not d.get("cbits") and (1 << (int(d["K"]) - int(d["rb"]))) == 256
               and dfma_per_amp(ops, int(d["rb"])) >= GROUPS_MIN_DFMA)
        if GROUPS_ONLY is not None:  # debugging: two groups for one descriptor only
            two = i == GROUPS_ONLY and not d.get("cbits")
        gen = kernel_source_2g if two else kernel_source
        if two:
            groups[i] = 2
        if (ld_xor or {}).get(i) or (st_keep or {}).get(i) or i in bcast:
            gen = kernel_source  # the one-group kernel carries the load XOR / store mask / broadcast
            groups.pop(i, None)
            body = gen("KNAME", d, ops, buf.coef, zi, sparse.get(i), (ld_xor or {}).get(i, 0),
                       (st_keep or {}).get(i), bcast.get(i))
        else:
            body = gen("KNAME", d, ops, buf.coef, zi, sparse.get(i))
        h = hashlib.sha1(body.encode()).hexdigest()[:16]
        name = f"{prefix}_{h}"
        srcs.append(body.replace("KNAME", name))
        names.append(name)
    _LAST_ZERO_INIT.clear()
    _LAST_ZERO_INIT.update(used)
    _LAST_GROUPS.clear()
    _LAST_GROUPS.update(groups)
    built = iter(compile_async(srcs, [n for n in names if n is not None], threads))
    slots = [None if n is None else next(built) for n in names]
    if lazy:
        return names, slots
    return names, [None if sl is None else sl.cubin() for sl in slots]


class KernelSlot:
    """A kernel being compiled in the background: cubin() blocks until its
    image exists (from this process's pool or from another process through
    the disk cache), so sweeps can launch while later sweeps compile."""

    def __init__(self, name: str, h: str, future):
        self.name, self.h, self.future = name, h, future

    def cubin(self) -> bytes:
        import time

        while True:
            if self.future.done():
                return self.future.result()
            hit = _cached(self.h)
            if hit is not None:
                return hit
            time.sleep(0.001)


_COMPILE_POOL = None


def compile_async(srcs: list, names: list, threads: int | None = None) -> list:
    """Submit the kernels to the compile pool in launch order (identical
    sources once); the processes of one node start at different offsets and
    share results through the disk cache."""
    global _COMPILE_POOL
    local = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    if _COMPILE_POOL is None:
        # the processes of one node compile at the same time: share the host cores
        n = threads or max(1, min(32, (os.cpu_count() or 4) // max(local, 1)))
        _COMPILE_POOL = ThreadPoolExecutor(max_workers=n, thread_name_prefix="svb-nvrtc")
    keys = [_key(src) for src in srcs]
    first = {}
    for i, h in enumerate(keys):
        first.setdefault(h, i)
    order = sorted(first.values())
    if local > 1 and order:  # rotate: rank r begins its share of the list, then wraps
        r = (lrank * len(order)) // local
        order = order[:1] + order[r:] + order[1:r] if r > 1 else order
    futs = {}
    for i in order:
        futs[keys[i]] = _COMPILE_POOL.submit(_compile, srcs[i], names[i])
    return [KernelSlot(names[i], keys[i], futs[keys[i]]) for i in range(len(srcs))]


def load_kernel(name: str, cubin: bytes, device_index: int):
    key = (name, device_index)
    k = _kernels.get(key)
    if k is None:
        lib = _native.load()
        handle = ctypes.c_void_p()
        _native.check(lib.svb_jit_load(cubin, name.encode(), ctypes.byref(handle)), "svb_jit_load")
        k = handle.value
        _kernels[key] = k
    return k
