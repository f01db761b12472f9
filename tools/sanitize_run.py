"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck):
interpreter sweeps (d <= 12), generated JIT sweeps (QFT-16 and QV-16 with
remaps between ranks on one GPU), sampling, compare and the layout kernels.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_14098_b200 import compare, gather, plan as planmod, run_plan, sample, scatter  # noqa: E402
from paper_2509_14098_b200 import workloads  # noqa: E402,F401

docs = json.load(gzip.open(ROOT / "tests/golden/grid.json.gz", "rt"))
states = dict(np.load(ROOT / "tests/golden/grid_states.npz"))
n = 0
for doc in docs[::40]:
    if doc["name"] not in states:
        continue
    plan = planmod.from_json(json.dumps(doc["plan"]))
    res = run_plan(plan, shots=64, seed=1)
    err = float(np.max(np.abs(res.state.blocks.cpu().numpy() - states[doc["name"]])))
    assert err < 1e-10, (doc["name"], err)
    n += 1
# JIT path at D >= 16: a 4-rank QFT-20 plan (co-resident relabels) and QV-20
for name in ("qft20_h18-12", "qv20_h18-12"):
    plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
    a = run_plan(plan, jit=True)
    dense = gather(a.state)
    b = run_plan(plan, initial=dense, jit=True)  # host initial state: identity start + upload path
    _ = compare(gather(b.state), dense)
    _ = sample(dense, 100, 3)
    _ = scatter(dense, plan, 0)
    from paper_2509_14098_b200 import executor

    _ = executor._gather_chunked(a.state, None)  # chunked host gather (svb_gather_bits)
    n += 2
# QV-20 from |0...0>: sparse support-only sweeps, two tile groups, sampling CDF walk
plan = planmod.load(str(ROOT / "plans" / "qv20_h18-12.json.gz"))
_ = run_plan(plan, shots=500, seed=5)
n += 1
torch.cuda.synchronize()
print(f"sanitize_run: {n} runs ok", flush=True)
