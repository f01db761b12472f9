"""Generate the committed golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py            # fixtures in tests/golden/
    python tests/golden/make_golden.py --plans    # + benchmark plans in plans/

Everything downstream (oracle pinning, GPU parity tests, bench.py) reads the
files written here and never imports the reference at run time.

Outputs
  gates.json            reference matrices / flags for every gate kind
  grid.json.gz          plans (reference JSON wire format) + stats for the
                        acceptance grid (test_acceptance.py:59-94 shape),
                        the reference's executor unit cases and a random
                        all-gate-kinds family
  grid_states.npz       final DistState.blocks of every grid case with d <= 10
  cfg1.json.gz / cfg1_fp.npz   QFT-20 on 4 simulated ranks (BASELINE cfg1):
                        plans + a fingerprint of the 2^20 final amplitudes
  ../../plans/*.json.gz benchmark plans (QFT-30..34, QV-30..34, QAOA-35, SUP-36)
"""

from __future__ import annotations

import argparse
import gzip
import itertools
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = Path(os.environ.get("SVPART_SRC", "/root/reference/pkg/src"))
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(ROOT))

from svpart import circuits, qasm  # noqa: E402  (the reference)
from svpart.executor import gather, run_plan  # noqa: E402
from svpart.gates import GATE_SIGNATURES, gate_tensor  # noqa: E402
from svpart.graph import build_graph  # noqa: E402
from svpart.partitioner import BudgetTooSmall, InvalidHierarchy, make_hierarchy, partition  # noqa: E402
from svpart.plan import lower, to_json  # noqa: E402

from paper_2509_14098_b200 import workloads  # noqa: E402  (QASM emitters only)


def plan_of(src: str, budgets):
    return lower(partition(build_graph(qasm.parse(src)), make_hierarchy(budgets)))


def mixed(d: int, seed: int = 0, n: int | None = None) -> str:
    """Random circuit over all 19 reference gate kinds (coverage family)."""
    rng = np.random.default_rng(seed * 7919 + 3)
    n = n if n is not None else 6 * d
    kinds = sorted(GATE_SIGNATURES)
    lines = ["OPENQASM 2.0;", 'include "qelib1.inc";', f"qreg q[{d}];"]
    for _ in range(n):
        k = kinds[int(rng.integers(0, len(kinds)))]
        npar, nq, _ = GATE_SIGNATURES[k]
        if nq > d:
            continue
        qs = rng.permutation(d)[:nq].tolist()
        ps = [repr(float(x)) for x in rng.uniform(-math.pi, math.pi, size=npar)]
        par = f"({','.join(ps)})" if npar else ""
        lines.append(f"{k}{par} " + ",".join(f"q[{x}]" for x in qs) + ";")
    return "\n".join(lines) + "\n"


def hierarchies(d: int, ranks: int):
    # same generator shape as test_acceptance.py:45-56
    g = ranks.bit_length() - 1
    top = d - g
    if top < 1:
        return
    yield [top]
    second = max(2, top - 2)
    if second <= top:
        yield [top, second]
        third = max(2, top - 4)
        if third <= second:
            yield [top, second, third]


def stats_doc(res) -> dict:
    return {"task_counts": res.stats.task_counts, "exchanges": res.stats.exchanges,
            "amps_moved": res.stats.amps_moved, "bytes_moved": res.stats.bytes_moved}


def gates_doc() -> dict:
    rng = np.random.default_rng(1)
    out = {}
    for kind, (npar, _, _) in sorted(GATE_SIGNATURES.items()):
        samples = [tuple(float(x) for x in rng.uniform(-4, 4, size=npar)) for _ in range(3)] if npar else [()]
        if npar:
            samples.append(tuple(0.0 for _ in range(npar)))  # e.g. rx(0) is diagonal
        for ps in samples:
            g = gate_tensor(kind, ps)
            m = np.asarray(g.matrix)
            out[f"{kind}{list(ps)}"] = {
                "kind": kind, "params": list(ps), "re": m.real.tolist(), "im": m.imag.tolist(),
                "is_diagonal": bool(g.is_diagonal), "controls": sorted(g.control_dims),
            }
    return out


def grid_cases():
    fams = sorted(circuits.FAMILIES)
    for fam, d, ranks in itertools.product(fams + ["mixed"], (4, 6, 8, 10, 12), (1, 2, 4, 8)):
        src = mixed(d, seed=d + ranks) if fam == "mixed" else circuits.generate(fam, d, seed=1)
        for budgets in hierarchies(d, ranks):
            yield f"{fam}-{d}-r{ranks}-{'_'.join(map(str, budgets))}", src, budgets
    # executor unit cases (test_executor.py)
    ghz3 = "qreg q[3];\nh q[0];\ncx q[0],q[1];\ncx q[1],q[2];\n"
    yield "ghz3-2", ghz3, [2]
    yield "ghz3-3", ghz3, [3]
    yield "ghz3-3_2", ghz3, [3, 2]
    yield "ghz4-2", "qreg q[4];\nh q[0];\ncx q[0],q[1];\ncx q[1],q[2];\ncx q[2],q[3];\n", [2]
    yield "x0-2", "qreg q[2];\nx q[0];\n", [2]
    yield "pass-3-2", "qreg q[3];\nh q[1];\nh q[2];\ncx q[1],q[2];\ncx q[0],q[1];\n", [2]
    for seed in range(40):  # test_executor.py:188-197 style random instances
        rng = np.random.default_rng(seed)
        d = int(rng.integers(4, 9))
        budgets = [int(rng.integers(2, d + 1))]
        if rng.integers(0, 2) and budgets[0] > 2:
            budgets.append(int(rng.integers(2, budgets[0] + 1)))
        fam = (sorted(circuits.FAMILIES) + ["mixed"])[seed % 8]
        src = mixed(d, seed) if fam == "mixed" else circuits.generate(fam, d, seed=seed)
        yield f"rand{seed}-{fam}-{d}-{'_'.join(map(str, budgets))}", src, budgets


def make_grid(out: Path) -> None:
    docs, states = [], {}
    skipped = 0
    for name, src, budgets in grid_cases():
        try:
            plan = plan_of(src, budgets)
        except (BudgetTooSmall, InvalidHierarchy):
            skipped += 1
            continue
        res = run_plan(plan)
        doc = {"name": name, "budgets": budgets, "qasm": src, "plan": json.loads(to_json(plan)),
               "stats": stats_doc(res)}
        docs.append(doc)
        if plan.d <= 10:
            states[name] = np.asarray(res.state.blocks)
            states[name + "::dense"] = gather(res.state)
    with gzip.open(out / "grid.json.gz", "wt") as fh:
        json.dump(docs, fh)
    np.savez_compressed(out / "grid_states.npz", **states)
    print(f"grid: {len(docs)} cases ({skipped} invalid-budget skips), {len(states) // 2} with states")


def make_cfg1(out: Path) -> None:
    src = circuits.qft(20)
    docs = {}
    fps = {}
    rng = np.random.default_rng(20)
    idx = np.sort(rng.choice(1 << 20, size=4096, replace=False))
    for budgets in ([18], [18, 12]):
        plan = plan_of(src, budgets)
        t0 = time.perf_counter()
        res = run_plan(plan)
        dt = time.perf_counter() - t0
        key = "_".join(map(str, budgets))
        docs[key] = {"plan": json.loads(to_json(plan)), "stats": stats_doc(res), "seconds": dt}
        flat = np.asarray(res.state.blocks).reshape(-1)
        fps[key + "::idx"] = idx
        fps[key + "::amps"] = flat[idx]
        fps[key + "::sum"] = np.array([flat.sum()])
        fps[key + "::wsum"] = np.array([(np.arange(flat.size) % 1009 * flat).sum()])
        fps[key + "::norm"] = np.array([np.vdot(flat, flat).real])
        print(f"cfg1 {budgets}: reference run_plan {dt:.2f} s")
    with gzip.open(out / "cfg1.json.gz", "wt") as fh:
        json.dump(docs, fh)
    np.savez_compressed(out / "cfg1_fp.npz", **fps)


# Benchmark-family plans whose sweeps run at real tile geometry (D > K = 12):
# fixed-bit predicates, per-tile slot tables and multi-row devices are then
# exercised against the reference itself.  (name, qasm generator, budgets,
# initial basis state or None)
FAMILY_CASES = [
    ("qv20_h18-12", lambda: workloads.quantum_volume(20, seed=20), [18, 12], None),
    ("qv22_h22-12", lambda: workloads.quantum_volume(22, seed=22), [22, 12], None),
    ("qv21_h20-12", lambda: workloads.quantum_volume(21, seed=21, depth=10), [20, 12], None),
    ("qaoa20_h18-12", lambda: workloads.qaoa_maxcut(20, seed=20, p=2), [18, 12], None),
    ("sup20_h19-12", lambda: workloads.random_supremacy(20, seed=20, depth=12), [19, 12], None),
    ("qft20_h19-12_x", lambda: workloads.qft(20), [19, 12], 0xB5A3D),
    ("qv20_h20-12_x", lambda: workloads.quantum_volume(20, seed=23, depth=8), [20, 12], 0x3C0F1),
]
FP_SAMPLES = 8192


def fingerprint(flat: np.ndarray, seed: int) -> dict:
    """Sampled amplitudes + weighted sums of the flat rank-block storage: a
    permutation of the storage changes them (the tests recompute them)."""
    rng = np.random.default_rng(seed)
    n = flat.size
    idx = np.sort(rng.choice(n, size=min(FP_SAMPLES, n), replace=False))
    w = np.exp(2j * np.pi * rng.random(n))
    return {"idx": idx, "amps": flat[idx], "sum": np.array([flat.sum()]),
            "wsum": np.array([(w * flat).sum()]), "norm": np.array([np.vdot(flat, flat).real])}


def make_families(out: Path) -> None:
    docs, fps = {}, {}
    for name, gen, budgets, x in FAMILY_CASES:
        src = gen()
        plan = plan_of(src, budgets)
        initial = None
        if x is not None:
            initial = np.zeros(1 << plan.d, dtype=np.complex128)
            initial[x] = 1.0
        t0 = time.perf_counter()
        res = run_plan(plan, initial=initial)
        dt = time.perf_counter() - t0
        docs[name] = {"plan": json.loads(to_json(plan)), "stats": stats_doc(res), "seconds": dt,
                      "initial_basis": x, "budgets": budgets, "fp_seed": len(docs) + 1}
        flat = np.asarray(res.state.blocks).reshape(-1)
        for k, v in fingerprint(flat, seed=len(docs)).items():
            fps[f"{name}::{k}"] = v
        print(f"family {name}: d={plan.d} g={plan.g} reference run_plan {dt:.1f} s", flush=True)
    with gzip.open(out / "families.json.gz", "wt") as fh:
        json.dump(docs, fh)
    np.savez_compressed(out / "families_fp.npz", **fps)


BENCH = [
    ("qft30_h30-12", lambda: workloads.qft(30), [30, 12]),
    ("qft31_h30-12", lambda: workloads.qft(31), [30, 12]),
    ("qft32_h30-12", lambda: workloads.qft(32), [30, 12]),
    ("qft33_h30-12", lambda: workloads.qft(33), [30, 12]),
    ("qft34_h33-12", lambda: workloads.qft(34), [33, 12]),
    ("qft34_h32-12", lambda: workloads.qft(34), [32, 12]),
    ("qft34_h31-12", lambda: workloads.qft(34), [31, 12]),
    ("qv30_h30-12", lambda: workloads.quantum_volume(30, seed=34), [30, 12]),
    ("qv34_h33-12", lambda: workloads.quantum_volume(34, seed=34), [33, 12]),
    ("qv34_h32-12", lambda: workloads.quantum_volume(34, seed=34), [32, 12]),
    ("qv34_h31-12", lambda: workloads.quantum_volume(34, seed=34), [31, 12]),
    ("qaoa35_h32-12", lambda: workloads.qaoa_maxcut(35, seed=35), [32, 12]),
    ("sup36_h33-12", lambda: workloads.random_supremacy(36, seed=36), [33, 12]),
    ("qft20_h18", lambda: workloads.qft(20), [18]),
    ("qft20_h18-12", lambda: workloads.qft(20), [18, 12]),
    ("qft24_h22-12", lambda: workloads.qft(24), [22, 12]),
    ("qft26_h23-12", lambda: workloads.qft(26), [23, 12]),
    ("qv20_h18-12", lambda: workloads.quantum_volume(20, seed=20), [18, 12]),
    ("qft22_h22-12", lambda: workloads.qft(22), [22, 12]),
    ("qft23_h23-12", lambda: workloads.qft(23), [23, 12]),
    ("qv22_h22-12", lambda: workloads.quantum_volume(22, seed=22), [22, 12]),
    ("qft28_h28-12", lambda: workloads.qft(28), [28, 12]),
    ("mirror_qv24_h22-12", lambda: workloads.mirror(workloads.quantum_volume(24, seed=5)), [22, 12]),
    ("mirror_qaoa24_h24-12", lambda: workloads.mirror(workloads.qaoa_maxcut(24, seed=6)), [24, 12]),
    ("mirror_sup24_h21-12", lambda: workloads.mirror(workloads.random_supremacy(24, seed=7)), [21, 12]),
    ("mirror_qv28_h28-12", lambda: workloads.mirror(workloads.quantum_volume(28, seed=8, depth=12)), [28, 12]),
    # multi-GPU full-size parity (sharded U U^dagger -> |0...0> checks in tools/dist_check.py)
    ("mirror_qv30_h29-12", lambda: workloads.mirror(workloads.quantum_volume(30, seed=9, depth=12)), [29, 12]),
    ("mirror_qv31_h29-12", lambda: workloads.mirror(workloads.quantum_volume(31, seed=10, depth=12)), [29, 12]),
    ("mirror_sup31_h29-12", lambda: workloads.mirror(workloads.random_supremacy(31, seed=11)), [29, 12]),
    ("mirror_qaoa31_h29-12", lambda: workloads.mirror(workloads.qaoa_maxcut(31, seed=12, p=2)), [29, 12]),
    # 8 ranks of 2^28 (world-8 remaps with m up to 3; eight processes can share one GPU)
    ("mirror_qv31_h28-12", lambda: workloads.mirror(workloads.quantum_volume(31, seed=14, depth=10)), [28, 12]),
    ("mirror_sup31_h28-12", lambda: workloads.mirror(workloads.random_supremacy(31, seed=15)), [28, 12]),
    ("mirror_qaoa31_h28-12", lambda: workloads.mirror(workloads.qaoa_maxcut(31, seed=16, p=2)), [28, 12]),
    # the exact QV-30 bench circuit inverted: forward + inverse from a random basis state on one GPU
    ("qv30inv_h30-12", lambda: workloads.inverse(workloads.quantum_volume(30, seed=34)), [30, 12]),
    # 34-qubit QV mirror on 2 GPUs (cfg3 shape, half depth each way): tools/dist_check.py --qv34
    ("mirror_qv34_h33-12", lambda: workloads.mirror(workloads.quantum_volume(34, seed=13, depth=17)), [33, 12]),
]


def make_plans(out: Path, force: bool = False) -> None:
    out.mkdir(exist_ok=True)
    mpath = out / "plans.json"
    meta = json.loads(mpath.read_text()) if mpath.exists() and not force else {}
    for name, gen, budgets in BENCH:
        if name in meta and (out / f"{name}.json.gz").exists():
            continue
        src = gen()
        t0 = time.perf_counter()
        plan = plan_of(src, budgets)
        dt = time.perf_counter() - t0
        with gzip.open(out / f"{name}.json.gz", "wt") as fh:
            fh.write(to_json(plan))
        fused = [t for t in plan.tasks if t.kind == "ApplyFused"]
        ex = [t for t in plan.tasks if t.kind == "Exchange"]
        meta[name] = {
            "d": plan.d, "g": plan.g, "budgets": budgets, "gates": len(qasm.parse(src).ops),
            "apply_fused": len(fused), "exchanges": [len(t.payload["swaps"]) for t in ex],
            "partition_seconds": round(dt, 3),
        }
        print(name, meta[name])
    (out / "plans.json").write_text(json.dumps(meta, indent=2, sort_keys=True) + "\n")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--plans", action="store_true", help="also write benchmark plans to plans/")
    ap.add_argument("--only-plans", action="store_true")
    ap.add_argument("--force", action="store_true", help="regenerate existing plans")
    ap.add_argument("--families", action="store_true", help="only the benchmark-family fingerprints")
    a = ap.parse_args()
    if a.families:
        make_families(HERE)
        sys.exit(0)
    if not a.only_plans:
        (HERE / "gates.json").write_text(json.dumps(gates_doc(), indent=1, sort_keys=True) + "\n")
        make_grid(HERE)
        make_cfg1(HERE)
        make_families(HERE)
    if a.plans or a.only_plans:
        make_plans(ROOT / "plans", a.force)
