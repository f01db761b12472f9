"""Per-sweep time of a plan on one GPU beside each sweep's FP64 work
(dense 4x4 / 2x2 FMAs per amplitude) and its HBM time at the copy peak:
which sweeps are HBM-bound, which FP64-bound."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2509_14098_b200 import executor, jit, plan as planmod, run_plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qv30_h30-12"
plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
for _ in range(2):
    run_plan(plan).wait()
executor.PROFILE_SWEEPS = True
prof = {}
for _ in range(3):
    r = run_plan(plan).wait()
    for di, lst in r.stats.sweep_profile.items():
        prof.setdefault(di, []).extend(ms for _, ms in lst)
comp = next(c for _, (pl, c) in executor._compile_cache.items() if pl is plan)
from paper_2509_14098_b200 import program as prog  # noqa: E402

hbm = 6546.2e9
rows = []
tot = tot_hbm = 0.0
for di in sorted(prof):
    ms = sum(prof[di]) / len(prof[di])
    nb = comp.desc_bytes[di]
    t_hbm = nb / hbm * 1e3
    rows.append((di, ms, t_hbm))
    tot += ms
    tot_hbm += max(t_hbm, 0)
print(f"{name}: {len(rows)} sweeps, {tot:.1f} ms of sweeps, HBM floor {tot_hbm:.1f} ms")
light = [r for r in rows if r[1] < 1.15 * r[2]]
print(f"  HBM-bound (within 15% of the HBM floor): {len(light)} sweeps, {sum(r[1] for r in light):.1f} ms")
for di, ms, th in rows:
    print(f"  sweep {di:3d}: {ms:7.2f} ms  hbm floor {th:6.2f} ms  ratio {ms / th:5.2f}")
