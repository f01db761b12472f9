"""Run one plan once on cuda:0 (for ncu: the k-th svb_jit launch is sweep k).

    ncu --set full -k regex:svb_jit_ --launch-skip K --launch-count 1 \\
        python tools/prof_sweep.py qv30_h30-12
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2509_14098_b200 import plan as planmod, run_plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qv30_h30-12"
plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
res = run_plan(plan)
torch.cuda.synchronize()
print(name, "sweeps", res.stats.sweeps, "launches", res.stats.kernel_launches)
