"""Run one plan N times (for ncu launch lists / full captures of k_sweep)."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2509_14098_b200 import plan as planmod, run_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--plan", default="qft30_h30-12")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
plan = planmod.load(str(ROOT / "plans" / f"{a.plan}.json.gz"))
for i in range(a.reps):
    r = run_plan(plan)
    torch.cuda.synchronize()
    print(i, "compute_ms", 1e3 * r.stats.compute_seconds, "sweeps", r.stats.sweeps, flush=True)
