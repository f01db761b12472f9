"""Distributed parity check: run plans over N processes (one GPU each, NCCL)
and compare the gathered state with the CPU oracle.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/dist_check.py [--quick]
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


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
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
    if me == 0:
        print(f"dist_check world={world}: {n} runs, {bad} mismatches", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


main()
