"""Stable file format of a compiled device program.

A plan compiled for one device (program.plan_device, with the generated
sweep kernels of jit.py) is written as a little-endian section file that a
native host reads without Python: native_host/svb_run.cpp loads it together
with the plan JSON (svpart/plan.py:171-201 wire format), validates the task
protocol like the reference executor, compiles and launches the kernels
through include/svb200.h and checks the norms.

    "SVBP" u32 version, then sections: 4-byte tag, u64 length, payload
    HEAD  i32 d, g, L, D, rows, n_fused, sparse, nsteps, ndescs, nkernels, unit
    BLOB  program blob (ops, coefficients, tables; prog.pack)
    DESC  ndescs x svb_sweep_desc (program.DESC_DTYPE, the C layout)
    STEP  nsteps x i32 {kind (0 sweeps, 1 exchange, 2 materialize), task id
          (-1 none), first descriptor, count, remote swaps}
    ALIA  n_fused x i32: slot whose sweep measured the norm (-1: carried)
    KERN  per descriptor: u32 len + kernel name, u32 len + CUDA source
    OPTS  u32 count, then u32 len + NVRTC option each
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from . import jit as jitmod, program as prog

MAGIC = b"SVBP"
VERSION = 1
KIND = {"sweeps": 0, "exchange": 1, "materialize": 2}


def _section(tag: bytes, payload: bytes) -> bytes:
    assert len(tag) == 4
    return tag + struct.pack("<Q", len(payload)) + payload


def export(plan, path: str | Path, zero_start: bool = True) -> Path:
    """Compile `plan` for one device holding every rank and write
    <path>.svbp (program) and <path>.plan.json (the plan wire format)."""
    from .plan import to_json

    path = Path(path)
    d, g = plan.d, plan.g
    geo = prog.DeviceGeometry(d=d, g=g, h=g, rank_base=0, pad_to=prog.RB)
    dp = prog.plan_device(plan, geo, rb=4, free_start=zero_start)
    sparse = prog.sparse_start(dp, geo.D, True) if zero_start else {}
    blob, descs, _ = prog.pack(dp.buf)
    srcs, names, groups = [], [], {}
    for i, dsc in enumerate(dp.buf.descs):
        ops = dp.buf.ops[dsc["op_begin"]: dsc["op_begin"] + dsc["op_count"]]
        zi = 0
        if i in sparse and sparse[i][0] is None:
            zi = 2
        elif i in sparse and sparse[i][0] == 0:
            zi = 1
        two = (jitmod.GROUPS and not dsc.get("cbits") and (1 << (int(dsc["K"]) - int(dsc["rb"]))) == 256
               and jitmod.dfma_per_amp(ops, int(dsc["rb"])) >= jitmod.GROUPS_MIN_DFMA)
        gen = jitmod.kernel_source_2g if two else jitmod.kernel_source
        body = gen("KNAME", dsc, ops, dp.buf.coef, zi, sparse.get(i))
        import hashlib

        name = "svb_jit_" + hashlib.sha1(body.encode()).hexdigest()[:16]
        srcs.append(body.replace("KNAME", name))
        names.append(name)
        if two:
            descs[i]["groups"] = 2
    alias = [dp.norm_alias.get(s, -1) for s in range(dp.n_fused)]
    steps = []
    for st in dp.steps:
        steps.append((KIND[st.kind], st.task_id if st.task_id is not None else -1, st.first, st.count,
                      len(st.swaps)))
    head = struct.pack("<11i", d, g, geo.L, geo.D, 1 << geo.h, dp.n_fused, 1 if sparse else 0, len(steps),
                       len(dp.buf.descs), len(srcs), 1)
    out = bytearray(MAGIC + struct.pack("<I", VERSION))
    out += _section(b"HEAD", head)
    out += _section(b"BLOB", np.ascontiguousarray(blob).tobytes())
    out += _section(b"DESC", descs.tobytes())
    out += _section(b"STEP", np.asarray(steps, dtype="<i4").reshape(-1, 5).tobytes())
    out += _section(b"ALIA", np.asarray(alias, dtype="<i4").tobytes())
    kern = bytearray()
    for nm, src in zip(names, srcs):
        b_nm, b_src = nm.encode(), src.encode()
        kern += struct.pack("<I", len(b_nm)) + b_nm + struct.pack("<I", len(b_src)) + b_src
    out += _section(b"KERN", bytes(kern))
    opts = bytearray(struct.pack("<I", len(jitmod.NVRTC_OPTS)))
    for o in jitmod.NVRTC_OPTS:
        opts += struct.pack("<I", len(o.encode())) + o.encode()
    out += _section(b"OPTS", bytes(opts))
    p_prog = path.with_suffix(".svbp")
    p_prog.write_bytes(bytes(out))
    path.with_suffix(".plan.json").write_text(to_json(plan))
    return p_prog


def read(path: str | Path) -> dict:
    """Parse a program file back (tests: the native host reads the same bytes)."""
    raw = Path(path).read_bytes()
    assert raw[:4] == MAGIC and struct.unpack("<I", raw[4:8])[0] == VERSION
    off, secs = 8, {}
    while off < len(raw):
        tag = raw[off:off + 4]
        (n,) = struct.unpack("<Q", raw[off + 4:off + 12])
        secs[tag.decode()] = raw[off + 12:off + 12 + n]
        off += 12 + n
    return secs
