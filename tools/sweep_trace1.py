"""Per-sweep times of one plan on one GPU (SVB200_TRACE=1), e.g. to see how
the sweep rate depends on the state size.

    SVB200_TRACE=1 python tools/sweep_trace1.py qft33_h30-12
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2509_14098_b200 import plan as planmod, run_plan  # noqa: E402

for name in sys.argv[1:]:
    plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
    for _ in range(2):
        res = run_plan(plan)
        del res
    res = run_plan(plan)
    torch.cuda.synchronize()
    tr = res.stats.trace
    n = 1 << plan.d
    print(f"{name}: {n * 16 / 2**30:.0f} GiB", flush=True)
    for (a, t0), (b, t1) in zip(tr[::2], tr[1::2]):
        print(f"  {a.replace(' start', ''):24s} {t1 - t0:8.2f} ms  {32 * n / (t1 - t0) / 1e9 * 1e3 / 1e3:7.0f} GB/s"
              if "sweep" in a and "-" not in a else f"  {a.replace(' start', ''):24s} {t1 - t0:8.2f} ms", flush=True)
    del res
