"""Sweep throughput vs grid size on one GPU: how much HBM rate the fused
sweeps keep when some SMs are left to a concurrent remap kernel."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2509_14098_b200 import plan as planmod, run_plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qft30_h30-12"
plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
for grid in (0, 132, 116, 100, 84):
    best = 1e9
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        res = run_plan(plan, grid_limit=grid)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
        del res
    print(f"{name} grid {grid or 148}: {best:.2f} ms", flush=True)
