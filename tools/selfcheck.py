"""Self-check run (what compute-sanitizer would be asked; it is closed on
this pool): every global index of the generated sweep kernels bounds-checked
with a trap (SVB200_JIT_CHECK=1), the state between NaN-patterned guard
bands verified after each run (SVB200_GUARD_AMPS), and every plan repeated
with different grid sizes -- a race in the barrier-light tile pipelines
(slot tables one tile ahead, mbarrier-tracked buffer rotation, two tile
groups, sparse zero tiles) would show as results that differ between grid
shapes.  Prints one line per plan; exits non-zero on any difference.

    SVB200_JIT_CHECK=1 SVB200_GUARD_AMPS=65536 python tools/selfcheck.py
"""
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_14098_b200 import executor, jit, plan as planmod, run_plan  # noqa: E402

assert jit.CHECK and executor.GUARD_AMPS, "run with SVB200_JIT_CHECK=1 SVB200_GUARD_AMPS=<n>"
fams = json.load(gzip.open(ROOT / "tests/golden/families.json.gz", "rt"))
plans = [(n, planmod.from_json(json.dumps(fams[n]["plan"]))) for n in ("qv20_h18-12", "qv21_h20-12", "qaoa20_h18-12",
                                                                       "sup20_h19-12")]
# qft22/qft28 from |0>: their last sweep is broadcast-merged into the one before
plans += [(n, planmod.load(str(ROOT / "plans" / f"{n}.json.gz")))
          for n in ("qft20_h18-12", "qft22_h22-12", "qft24_h22-12", "qft28_h28-12", "mirror_qv24_h22-12")]
bad = 0
for name, plan in plans:
    ref = None
    for grid in (0, 37, 5):
        for initial in (None, "basis"):
            init = None
            if initial:
                init = torch.zeros((1 << plan.g, 1 << (plan.d - plan.g)), dtype=torch.complex128, device="cuda")
                init[0, 3] = 1.0
            res = run_plan(plan, grid_limit=grid, initial=init)
            got = res.state.blocks.cpu().numpy()
            torch.cuda.synchronize()
            key = initial or "zero"
            if ref is None:
                ref = {}
            if key not in ref:
                ref[key] = got
            elif not np.array_equal(ref[key], got):
                bad += 1
                print("MISMATCH", name, "grid", grid, key, flush=True)
    print(name, "grids 148/37/5 x starts |0>,|3>: bit-identical, bounds and guards clean", flush=True)
print(f"selfcheck: {len(plans)} plans, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
