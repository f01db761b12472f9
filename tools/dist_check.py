"""Distributed parity check: run plans over N processes (one GPU each, NCCL)
and compare the gathered state with the CPU oracle.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/dist_check.py [--quick] [--scale] [--qft34] [--qv34]
                                                                             [--colocate]

--colocate runs every process on cuda:0 with a gloo control plane (the
inter-process peer remap then runs between processes sharing one GPU).
"""
import gzip
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2509_14098_b200 import gather, plan as planmod, run_plan  # noqa: E402


def qft_closed_form_err(state, x: int) -> float:
    """max |amp - 2^-d/2 exp(-2 pi i x y / 2^d)| over this process's shard,
    all-reduced; chunked so a 2^33-amplitude shard needs no index array."""
    d, L = state.d, state.d - state.g
    layout = state.layouts[state.phase]
    flat = state.blocks.reshape(-1)
    n = flat.numel()
    base = state.rank_base << L
    mask = (1 << d) - 1
    lo_bits = min(d, 20)
    xl, xh = x & ((1 << lo_bits) - 1), x >> lo_bits
    err = torch.zeros((), dtype=torch.float64, device=flat.device)
    chunk = 1 << 24
    for off in range(0, n, chunk):
        f = torch.arange(off, min(off + chunk, n), device=flat.device, dtype=torch.int64) + base
        y = torch.zeros_like(f)
        for q in range(d):  # storage bit d-1-layout[q] -> basis bit d-1-q
            y |= ((f >> (d - 1 - layout[q])) & 1) << (d - 1 - q)
        # x*y mod 2^d without int64 overflow: split x into low/high parts
        r = ((y * xl) + (((y * xh) & ((1 << max(d - lo_bits, 0)) - 1)) << lo_bits)) & mask
        exp = torch.exp(-2j * np.pi * r.to(torch.float64) / (1 << d)) / 2 ** (d / 2)
        err = torch.maximum(err, (flat[off:off + f.numel()] - exp).abs().max())
    dist.all_reduce(err, op=dist.ReduceOp.MAX)
    return float(err.item())


def basis_blocks(plan, x: int, rank_base: int, rows: int, device) -> torch.Tensor:
    """This process's phase-0 rank blocks of the basis state |x> (device tensor)."""
    d, g = plan.d, plan.g
    L = d - g
    layout = plan.layout_phases[0]
    f = 0
    for q in range(d):
        if (x >> (d - 1 - q)) & 1:
            f |= 1 << (d - 1 - layout[q])
    blocks = torch.zeros((rows, 1 << L), dtype=torch.complex128, device=device)
    if rank_base <= f >> L < rank_base + rows:
        blocks[(f >> L) - rank_base, f & ((1 << L) - 1)] = 1.0
    return blocks


def scale_checks(me, world):
    """Full-size parity through size-independent properties, with no gather:
    QFT of a basis state against its closed form, and sharded compare()."""
    from paper_2509_14098_b200 import compare, fidelity

    bad = n = 0
    lg = world.bit_length() - 1
    # a basis state (dense sweeps, the NVLink remap) and |0...0> (sparse sweeps;
    # the first remap is localized: every process replicates the prefix)
    names = [(f"qft{30 + lg}_h30-12", 0x2B3C5D1 << lg | 1), (f"qft{30 + lg}_h30-12", 0)]
    if "--qft34" in sys.argv:
        names.append((f"qft34_h{34 - lg}-12", 0))
    for name, x in names:
        plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
        if "--colocate" in sys.argv:  # all processes share one GPU's memory
            from paper_2509_14098_b200 import comm

            comm.release_arenas()
            torch.cuda.empty_cache()
        rows = (1 << plan.g) // world
        # processes sharing one GPU keep the initial blocks in host memory
        init = basis_blocks(plan, x, me * rows, rows, "cpu" if "--colocate" in sys.argv else "cuda") if x else None
        res = run_plan(plan, initial=init)
        del init
        err = qft_closed_form_err(res.state, x)
        n += 1
        bad += err > 1e-10
        if me == 0:
            print(name, "x", hex(x), "closed-form err", err, "remaps", len(res.stats.exchanges), flush=True)
        del res
    # mirror circuits U U^dagger over several GPUs (QV with 4-5 remaps, supremacy): every
    # amplitude must return to the start |x>, checked shard by shard
    mirrors = ["mirror_qv30_h29-12", "mirror_qv31_h29-12", "mirror_sup31_h29-12", "mirror_qaoa31_h29-12",
               # 8 ranks: m = 3 remaps (every partner of a rank at world 8)
               "mirror_qv31_h28-12", "mirror_sup31_h28-12", "mirror_qaoa31_h28-12"]
    if "--qv34" in sys.argv:  # 34 qubits: 2 GPUs of 128 GiB each
        mirrors.append("mirror_qv34_h33-12")
    for name in mirrors:
        plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
        if (1 << plan.g) < world:
            continue
        # return the pooled buffers of earlier runs first (a 128 GiB QFT-34
        # arena and the mirrors' own would not fit together)
        from paper_2509_14098_b200 import comm

        comm.release_arenas()
        torch.cuda.empty_cache()
        # U U^dagger |x> = |x> from a random basis state: every amplitude and
        # its storage position are checked (|0...0> would hide a wrong relabel
        # or final materialisation: it is invariant under bit permutations)
        x = (0x9E3779B97F4A7C15 * (len(name) + 7)) & ((1 << plan.d) - 1)
        rows = (1 << plan.g) // world
        init = basis_blocks(plan, x, me * rows, rows, "cpu" if "--colocate" in sys.argv else "cuda")
        res = run_plan(plan, initial=init)
        del init
        L = plan.d - plan.g
        fin = res.state.layouts[res.state.phase]
        f = 0
        for q in range(plan.d):
            if (x >> (plan.d - 1 - q)) & 1:
                f |= 1 << (plan.d - 1 - fin[q])
        flat = res.state.blocks.reshape(-1)
        local = f - (res.state.rank_base << L)
        if 0 <= local < flat.numel():
            flat[local] -= 1.0  # the one amplitude that must be 1
        err = torch.zeros(1, dtype=torch.float64, device=flat.device)
        for off in range(0, flat.numel(), 1 << 26):  # chunked: no full-size temporaries
            err = torch.maximum(err, flat[off:off + (1 << 26)].abs().max().reshape(1))
        dist.all_reduce(err, op=dist.ReduceOp.MAX)
        n += 1
        bad += float(err.item()) > 1e-10
        if me == 0:
            print(name, f"mirror |x> (x={x:#x}) err", float(err.item()), "remaps", len(res.stats.exchanges),
                  "ms", round(1e3 * (res.stats.compute_seconds + res.stats.exchange_seconds), 1), flush=True)
        del res, flat
    # sharded compare / fidelity vs the gathered reference compare
    plan = planmod.load(str(ROOT / "plans" / "qft20_h18-12.json.gz"))
    if (1 << plan.g) >= world:
        rng = np.random.default_rng(17)
        vs = []
        for _ in range(2):
            v = rng.normal(size=1 << plan.d) + 1j * rng.normal(size=1 << plan.d)
            vs.append(v / np.linalg.norm(v))
        sa, sb = (run_plan(plan, initial=v).state for v in vs)
        got, fid = compare(sa, sb), fidelity(sa, sb)
        ga, gb = gather(sa), gather(sb)
        want = orc.compare(ga, gb)
        wfid = abs(np.vdot(ga, gb)) ** 2
        same = compare(sa, sa)
        n += 1
        # CUDA's hypot may differ from libm's by an ulp: allow a few ulps
        ok = abs(got - want) <= 1e-14 * want and abs(fid - wfid) < 1e-12 and same == 0.0
        bad += not ok
        if me == 0:
            print("sharded compare", got, "reference", want, "fidelity", fid, wfid, "self", same, flush=True)
        # sharded device sampling vs numpy's Generator.choice on the gathered state
        for seed in (3, 4):
            hist = run_plan(plan, initial=vs[0], shots=5000, seed=seed).histogram
            p = np.abs(ga) ** 2
            outc = np.random.default_rng(seed).choice(len(ga), size=5000, p=p / p.sum())
            vals, cnts = np.unique(outc, return_counts=True)
            want_h = {format(int(v), f"0{plan.d}b"): int(c) for v, c in zip(vals, cnts)}
            n += 1
            bad += hist != want_h
            if me == 0:
                print("sharded sample seed", seed, "identical to numpy:", hist == want_h, flush=True)
    return n, bad


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "--colocate" in sys.argv:
        # every process on cuda:0 (the driver's GPU test box has one GPU):
        # the peer-memory remap still maps the other processes' state with
        # CUDA IPC and orders the swaps with flag words; NCCL refuses two
        # ranks on one device, so the control plane is gloo
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world = dist.get_world_size()
    me = dist.get_rank()
    docs = json.load(gzip.open(ROOT / "tests/golden/grid.json.gz", "rt"))
    states = dict(np.load(ROOT / "tests/golden/grid_states.npz"))
    quick = "--quick" in sys.argv
    if quick:
        docs = docs[::10]
    n = bad = 0
    for doc in docs:
        if doc["name"] not in states or (1 << doc["plan"]["g"]) < world:
            continue
        plan = planmod.from_json(json.dumps(doc["plan"]))
        for jit in (False, True) if plan.d >= 8 else (False,):
            res = run_plan(plan, jit=jit)
            dense = gather(res.state)
            err = float(np.max(np.abs(dense - states[doc["name"] + "::dense"])))
            n += 1
            if err > 1e-10:
                bad += 1
                if me == 0:
                    print("MISMATCH", doc["name"], "jit", jit, err, flush=True)
    # larger plans with real exchanges
    for name in ["qft20_h18-12", "qft24_h22-12"] if quick else ["qft20_h18-12", "qv20_h18-12", "qft24_h22-12"]:
        plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
        if (1 << plan.g) < world:
            continue
        t0 = time.perf_counter()
        res = run_plan(plan)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        dense = gather(res.state)
        if me == 0:
            ref, _ = orc.run_plan(plan, backend="c", nthreads=8)
            err = float(np.max(np.abs(dense - orc.gather(ref, plan.layout_phases[-1], plan.d))))
            print(name, "world", world, "err", err, "exchange_ms", 1e3 * res.stats.exchange_seconds,
                  "wall_s", round(dt, 3), flush=True)
            if err > 1e-10:
                bad += 1
        n += 1
    # initial states: the reference's dense vector, and this process's own
    # phase-0 rank blocks (the distributed form)
    for name in ["qft20_h18-12", "qv20_h18-12"]:
        plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
        if (1 << plan.g) < world:
            continue
        rng = np.random.default_rng(11)
        v = rng.normal(size=1 << plan.d) + 1j * rng.normal(size=1 << plan.d)
        v /= np.linalg.norm(v)
        ref_blocks, _ = orc.run_plan(plan, backend="c", nthreads=8, initial=v)
        want = orc.gather(ref_blocks, plan.layout_phases[-1], plan.d)
        rows = (1 << plan.g) // world
        mine = orc.scatter(v, plan.layout_phases[0], plan.d, plan.g)[me * rows:(me + 1) * rows]
        for form, init in (("dense", v), ("blocks", torch.from_numpy(np.ascontiguousarray(mine)))):
            dense = gather(run_plan(plan, initial=init).state)
            err = float(np.max(np.abs(dense - want)))
            n += 1
            if me == 0:
                print(name, "initial", form, "err", err, flush=True)
            if err > 1e-10:
                bad += 1
    if "--quick" not in sys.argv or "--scale" in sys.argv:
        n2, bad2 = scale_checks(me, world)
        n += n2
        bad += bad2
    if me == 0:
        print(f"dist_check world={world}: {n} runs, {bad} mismatches", flush=True)
    from paper_2509_14098_b200 import comm

    freed = comm.release_arenas()
    if me == 0:
        print(f"released {freed} pooled state buffers", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


main()
