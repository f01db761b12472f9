"""Numpy emulator of the fused sweep kernel (csrc/sweep.cu) -- tests only.

Executes a compiled program (paper_2509_14098_b200.program.pack output)
exactly as the kernel does -- same tile origins, shared-memory swizzle, stage
mappings, register slots, predicates and phase tables -- but vectorised over
threads with numpy.  Comparing it with the oracle validates the host
compiler on machines without a GPU; the GPU parity tests then validate the
kernel against the same oracle.
"""

from __future__ import annotations

import numpy as np

from paper_2509_14098_b200 import program as prog



def _dep(vals: np.ndarray, bits) -> np.ndarray:
    out = np.zeros_like(vals, dtype=np.int64)
    for i, b in enumerate(bits):
        out |= ((vals >> i) & 1) << b
    return out


def _xor_img(vals: np.ndarray, imgs) -> np.ndarray:
    out = np.zeros_like(vals, dtype=np.int64)
    for i, s in enumerate(imgs):
        out ^= np.where((vals >> i) & 1, s, 0)
    return out


def run_sweeps(state: np.ndarray, descs, parts, norms: np.ndarray | None = None, sparse=None,
               ld_xor=None, st_keep=None) -> None:
    """In-place on the flat device state (length 2^D).

    sparse: per descriptor (support, full_out) or None (program.sparse_start);
    a sparse sweep computes only live tiles, zero-fills loads outside the
    support (the unit vector when the support is empty) and writes zeros
    over the dead tiles only when full_out, as the generated kernel does."""
    ops_all, coef, tab, cterms, cofs_all = (parts[k] for k in ("ops", "coef", "tab", "cterms", "cofs"))
    cofs_base = 0
    for di, d in enumerate(descs):
        sp = sparse[di] if sparse is not None else None
        lx = (ld_xor[di] or 0) if ld_xor is not None else 0
        keep = st_keep[di] if st_keep is not None else None
        K, D = int(d["K"]), int(d["D"])
        RB = int(d["rb"])
        NR = 1 << RB
        NT = 1 << (K - RB)
        tin = [int(x) for x in d["tin"][:K]]
        sw = [int(x) for x in d["sw"][:K]]
        st_dev = [int(x) for x in d["st_dev"][:K]]
        st_sw = [int(x) for x in d["st_sw"][:K]]
        st_flip = int(d["st_flip"])
        nct = int(d["nctab"])
        ops = ops_all[int(d["op_begin"]): int(d["op_begin"]) + int(d["op_count"])]
        ci = (int(d["cofs_off"]) - int(parts["cofs_base"])) // 4
        cofs = cofs_all[ci: ci + nct + 1]
        fbits = [b for b in range(D) if b not in tin]
        c_all = np.arange(1 << K, dtype=np.int64)
        ld_dev = _dep(c_all, tin)
        ld_s = _xor_img(c_all, sw)
        st_d = _dep(c_all, st_dev) ^ st_flip
        st_s = _xor_img(c_all, st_sw)
        tix = np.arange(NT, dtype=np.int64)
        nrm = 0.0
        for tile_id in range(1 << (D - K)):
            base = 0
            for i, b in enumerate(fbits):
                if (tile_id >> i) & 1:
                    base |= 1 << b
            if sp is not None:
                supp, full_out = sp
                if supp is None or base & ~supp:  # dead tile
                    if full_out:
                        state[base | ld_dev] = 0.0
                    continue
            ctab = np.ones(max(nct, 1), dtype=np.complex128)
            for i in range(nct):
                for q in range(int(cofs[i]), int(cofs[i + 1])):
                    ct = cterms[q]
                    if (base & int(ct["mask"])) == int(ct["mask"]):
                        ctab[i] *= complex(ct["re"], ct["im"])
            tile = np.empty(1 << K, dtype=np.complex128)
            if sp is None:
                tile[ld_s] = state[base | ld_dev]
            elif sp[0] == 0:  # synthesised |0...0>
                tile[ld_s] = np.where((base | ld_dev) == 0, 1.0 + 0j, 0j)
            else:  # zero-filled outside the support (a folded localize reads region alpha)
                pos = base | ld_dev
                tile[ld_s] = np.where((pos & ~sp[0]) == 0, state[pos ^ lx], 0j)
            x = None
            J = None
            dev_base = None
            for op in ops:
                kind = int(op["kind"])
                if kind == prog.OP_STAGE:
                    if x is not None:
                        tile[J] = x
                    rm = int(op["rmask"])
                    regs = [k for k in range(K) if (rm >> k) & 1]
                    if int(op["flags"]) & prog.F_TORDER:  # planner-chosen thread-bit order
                        comp = prog.unpack_order(int(op["pval"]), K - len(regs))
                    else:
                        comp = [k for k in range(K) if not (rm >> k) & 1]
                    jt = _dep(tix, comp)
                    jv = _dep(np.arange(NR, dtype=np.int64), regs)
                    jj = jt[:, None] | jv[None, :]
                    J = _img(jj, sw)
                    x = tile[J].copy()
                    dev_base = base | _devmap(jt, tin)
                    continue
                pred = (dev_base & int(op["pmask"])) == int(op["pval"])
                if not pred.any():
                    continue
                a = int(op["a"])
                cf = int(op["coef"])
                cm, cv = int(op["rmask"]), int(op["b"])
                xs = x.copy()
                if kind in (prog.OP_H, prog.OP_U1, prog.OP_PH):
                    has_phase = kind == prog.OP_PH or (int(op["flags"]) & prog.F_PHASE)
                    if has_phase:
                        ph = cf if kind == prog.OP_PH else cf + 4
                        p = np.full(NT, coef[ph], dtype=np.complex128)
                        if int(op["ctab"]) >= 0:
                            p = p * ctab[int(op["ctab"])]
                        if int(op["tab"]) >= 0:
                            p = p * tab[int(op["tab"]) + tix]
                        if int(op["tf"]) >= 0:
                            for i in range(K - RB):
                                p = np.where((tix >> i) & 1, p * ctab[int(op["tf"]) + i], p)
                        nt = (int(op["flags"]) >> prog.F_PREG_SHIFT) & 0xF
                        for v in range(NR):
                            if not (v >> a) & 1:
                                continue
                            q = p.copy()
                            for s in range(RB):
                                if s != a and (v >> s) & 1 and (nt >> s) & 1:
                                    q = q * coef[ph + 1 + s]
                            xs[:, v] = xs[:, v] * q
                    if kind == prog.OP_H:
                        for v in range(NR):
                            if (v >> a) & 1 or (v & cm) != cv:
                                continue
                            x0, x1 = xs[:, v].copy(), xs[:, v | (1 << a)].copy()
                            xs[:, v], xs[:, v | (1 << a)] = x0 + x1, x0 - x1
                    elif kind == prog.OP_U1:
                        m00, m01, m10, m11 = coef[cf:cf + 4]
                        for v in range(NR):
                            if (v >> a) & 1 or (v & cm) != cv:
                                continue
                            x0, x1 = xs[:, v].copy(), xs[:, v | (1 << a)].copy()
                            xs[:, v], xs[:, v | (1 << a)] = m00 * x0 + m01 * x1, m10 * x0 + m11 * x1
                elif kind == prog.OP_X:
                    for v in range(NR):
                        if (v >> a) & 1 or (v & cm) != cv:
                            continue
                        x0, x1 = xs[:, v].copy(), xs[:, v | (1 << a)].copy()
                        xs[:, v], xs[:, v | (1 << a)] = x1, x0
                elif kind == prog.OP_U2:
                    b = int(op["b"])
                    M = coef[cf:cf + 16].reshape(4, 4)
                    for v in range(NR):
                        if (v >> a) & 1 or (v >> b) & 1:
                            continue
                        idx = [v, v | (1 << b), v | (1 << a), v | (1 << a) | (1 << b)]
                        y = M @ xs[:, idx].T
                        xs[:, idx] = y.T
                elif kind == prog.OP_PHALL:
                    p = np.full(NT, coef[cf], dtype=np.complex128)
                    if int(op["ctab"]) >= 0:
                        p = p * ctab[int(op["ctab"])]
                    if int(op["tab"]) >= 0:
                        p = p * tab[int(op["tab"]) + tix]
                    if int(op["tf"]) >= 0:
                        for i in range(K - RB):
                            p = np.where((tix >> i) & 1, p * ctab[int(op["tf"]) + i], p)
                    xs = xs * p[:, None]
                elif kind == prog.OP_SCALE:
                    xs = xs * coef[cf]
                x = np.where(pred[:, None], xs, x)
            if x is not None:
                tile[J] = x
            vals = tile[st_s]
            nrm += float(np.sum(np.abs(vals) ** 2))
            if keep is None:
                state[base | st_d] = vals
            else:  # only this process's region of a localized remap is stored
                sel = ((base | st_d) & keep[0]) == keep[1]
                state[(base | st_d)[sel]] = vals[sel]
        slot = int(d["norm_slot"])
        if norms is not None and slot >= 0:
            norms[slot] += nrm
        cofs_base += nct + 1


def _img(jj: np.ndarray, sw) -> np.ndarray:
    out = np.zeros_like(jj)
    for k, s in enumerate(sw):
        out ^= np.where((jj >> k) & 1, s, 0)
    return out


def _devmap(jt: np.ndarray, tin) -> np.ndarray:
    out = np.zeros_like(jt)
    for k, b in enumerate(tin):
        out |= ((jt >> k) & 1) << b
    return out


LAST_MERGES = 0  # broadcast merges applied by the last emulate_plan (all devices)


def _broadcast(state: np.ndarray, bc, keep) -> None:
    """The merged store of executor._broadcast_merges: every value sweep j
    stored (region `keep` of the masked bits, F bits otherwise clear) is
    written, times its combination's constants, at each combination of F."""
    fmask, copies = bc[0], bc[1]
    km, kv = keep if keep is not None else (0, 0)
    idx = np.arange(state.size, dtype=np.int64)
    sel = idx[((idx & (fmask & ~km)) == 0) & ((idx & km) == kv)]
    v = state[sel].copy()
    base = sel & ~fmask
    bits = [b for b in range(fmask.bit_length()) if (fmask >> b) & 1]
    for j in range(1 << len(bits)):
        f = sum(1 << bits[i] for i in range(len(bits)) if (j >> i) & 1)
        val = np.zeros_like(v)
        if f in copies:
            val = v.copy()
            for c in copies[f]:
                val = val * c
        state[base | f] = val


def emulate_plan(plan, world: int = 1, check_layout: bool = True, rb: int = prog.RB, stable: bool = False,
                 sparse: bool = False, kmax: int = prog.KMAX, localize: bool = False, fold: bool = True,
                 merge: bool = False):
    """Run a plan through the compiled device programs of `world` devices.

    Each device gets its own program (plan_device with its rank range);
    exchanges are applied as the physical bit swaps the schedule names, on
    the concatenation of all devices' rows.  Returns the (2^g, 2^L) blocks.
    """
    d, g = plan.d, plan.g
    L = d - g
    nr = 1 << g
    rows = nr // world
    h = rows.bit_length() - 1
    progs, parts = [], []
    replicate = False
    if localize and sparse and world > 1:  # decided on the unit-holding process, as the executor does
        geo0 = prog.DeviceGeometry(d=d, g=g, h=h, rank_base=0, pad_to=prog.RB)
        replicate = prog.localize_applies(prog.plan_device(plan, geo0, rb=rb, stable_threads=stable, kmax=kmax),
                                          geo0.D, world, h)
    for w in range(world):
        geo = prog.DeviceGeometry(d=d, g=g, h=h, rank_base=w * rows, pad_to=prog.RB)
        dp = prog.plan_device(plan, geo, rb=rb, stable_threads=stable, kmax=kmax, replicate_prefix=replicate)
        blob, descs, p = prog.pack(dp.buf)
        progs.append((geo, dp, descs, p))
    D = progs[0][0].D
    # every device must derive the same layout schedule
    if check_layout:
        for geo, dp, _, _ in progs[1:]:
            assert [(s.kind, s.task_id, s.swaps) for s in dp.steps] == \
                [(s.kind, s.task_id, s.swaps) for s in progs[0][1].steps]
    states = [np.zeros(1 << D, dtype=np.complex128) for _ in range(world)]
    states[0][0] = 1.0
    bc_of = []  # per device: broadcast merges (executor._broadcast_merges)
    sp_of, lx_of, keep_of = [], [], []  # per device: descriptor -> (support, full_out) / load XOR / store mask
    for w, (geo, dp, descs, p) in enumerate(progs):
        sp = prog.sparse_start(dp, D, w == 0 or replicate) if sparse else {}
        if replicate and fold:
            from paper_2509_14098_b200.executor import _fold_localize, _prefix_store_masks

            lx_of.append(_fold_localize(dp, geo, sp))
            keep_of.append(_prefix_store_masks(dp, geo, sp))
        else:
            lx_of.append({})
            keep_of.append({})
        if sp:  # unwritten memory: any read outside the support would poison the result
            states[w][:] = np.nan
        sp_of.append(sp)
        if merge and sp:
            from paper_2509_14098_b200.executor import _broadcast_merges

            bc_of.append(_broadcast_merges(dp, geo, sp, lx_of[-1], keep_of[-1], {}))
        else:
            bc_of.append({})
    global LAST_MERGES
    LAST_MERGES = sum(len(b) for b in bc_of)
    norms = np.zeros(max(progs[0][1].n_fused, 1))
    steps = {s.task_id: s for s in progs[0][1].steps}
    for task in plan.tasks:
        st = steps.get(task.id)
        if task.kind == "ApplyFused":
            slot = sum(1 for t in plan.tasks[: plan.tasks.index(task)] if t.kind == "ApplyFused")
            for w, (geo, dp, descs, p) in enumerate(progs):
                sw = {s.task_id: s for s in dp.steps}[task.id]
                if not bc_of[w]:
                    run_sweeps(states[w], descs[sw.first: sw.first + sw.count], p, norms,
                               [sp_of[w].get(i) for i in range(sw.first, sw.first + sw.count)],
                               [lx_of[w].get(i) for i in range(sw.first, sw.first + sw.count)],
                               [keep_of[w].get(i) for i in range(sw.first, sw.first + sw.count)])
                    continue
                for i in range(sw.first, sw.first + sw.count):
                    if i - 1 in bc_of[w]:
                        continue  # merged into the sweep before it
                    run_sweeps(states[w], descs[i:i + 1], p, None, [sp_of[w].get(i)], [lx_of[w].get(i)],
                               [keep_of[w].get(i)])
                    if i in bc_of[w]:
                        _broadcast(states[w], bc_of[w][i], keep_of[w].get(i))
            if st.count == 0 and slot not in progs[0][1].norm_alias:
                norms[slot] = norms[slot - 1] if slot else 1.0  # |0...0> (maybe not materialised yet)
        elif task.kind == "Exchange" and st.kind == "localize":
            # every device moves region alpha (its id bits) of its replica to region 0
            # (unless the next sweep reads it through a load XOR)
            for w in range(world):
                if {s_.task_id: s_ for s_ in progs[w][1].steps}[task.id].folded:
                    continue
                me = w
                alpha, lbs = 0, []
                for ib, lb in st.swaps:
                    alpha = (alpha << 1) | ((me >> (ib - h)) & 1)
                    lbs.append(lb)
                if alpha:
                    m = len(lbs)
                    idx = np.arange(1 << D, dtype=np.int64)
                    sel = np.zeros_like(idx)
                    for i, lb in enumerate(lbs):
                        sel |= ((idx >> lb) & 1) << (m - 1 - i)
                    dst = idx[sel == 0]
                    src = dst.copy()
                    for i, lb in enumerate(lbs):
                        if (alpha >> (m - 1 - i)) & 1:
                            src |= 1 << lb
                    states[w][dst] = states[w][src]
        elif task.kind == "Exchange":
            # global index = device * 2^(L+h) + row * 2^L + local
            full = np.concatenate([s[: rows << L] for s in states])
            nb = (world.bit_length() - 1) + h + L
            x = full.reshape((2,) * nb)
            for ib, lb in st.swaps:
                u = L + ib
                x = np.swapaxes(x, nb - 1 - u, nb - 1 - lb)
            full = np.ascontiguousarray(x).reshape(-1)
            for w in range(world):
                states[w][: rows << L] = full[w * (rows << L):(w + 1) * (rows << L)]
    mat = steps.get(None)
    if mat is not None:
        for w, (geo, dp, descs, p) in enumerate(progs):
            run_sweeps(states[w], descs[mat.first: mat.first + mat.count], p, None,
                       [sp_of[w].get(i) for i in range(mat.first, mat.first + mat.count)],
                       [lx_of[w].get(i) for i in range(mat.first, mat.first + mat.count)])
    blocks = np.concatenate([s[: rows << L] for s in states]).reshape(nr, 1 << L)
    alias = progs[0][1].norm_alias
    norms = np.array([norms[alias.get(i, i)] for i in range(len(norms))])
    return blocks, norms
