"""Time of run_plan(shots=...) beside run_plan alone on one GPU (QFT-30 and
QV-30): the cost of numpy-identical sampling at full size."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2509_14098_b200 import plan as planmod, run_plan  # noqa: E402

for name in ("qft30_h30-12", "qv30_h30-12"):
    plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
    for _ in range(2):
        run_plan(plan, shots=1000, seed=1).wait()
    torch.cuda.synchronize()
    for shots in (0, 1000, 1000000):
        ts = []
        for rep in range(3):
            t0 = time.perf_counter()
            r = run_plan(plan, shots=shots or None, seed=7 + rep).wait()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            del r
        print(f"{name} shots={shots}: {1e3 * min(ts):.1f} ms (min of 3, wall)", flush=True)
