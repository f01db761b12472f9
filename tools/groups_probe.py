"""Which sweep's two-group kernel differs from its one-group kernel: runs the
plan once with one-group kernels, then once per descriptor with only that
descriptor in two-group form (SVB200_JIT_GROUPS_ONLY), each in a fresh
process, and compares the final blocks bit for bit."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
name = sys.argv[1]
dense = "--dense" in sys.argv
code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {str(ROOT)!r})
from paper_2509_14098_b200 import plan as planmod, run_plan
plan = planmod.load({str(ROOT / 'plans')!r} + '/{name}.json.gz')
r = run_plan(plan)
np.save(sys.argv[1], r.state.blocks.cpu().numpy())
print('sweeps', r.stats.sweeps)
"""
base = dict(os.environ, SVB200_JIT_GROUPS="0")
if dense:
    base["SVB200_SPARSE_START"] = "0"
r = subprocess.run([sys.executable, "-c", code, "/tmp/ref.npy"], env=base, capture_output=True, text=True, timeout=300)
print(r.stdout.strip(), r.stderr[-300:])
n = int(r.stdout.split()[-1])
import numpy as np  # noqa: E402

ref = np.load("/tmp/ref.npy")
for i in range(n):
    env = dict(base, SVB200_JIT_GROUPS="1", SVB200_JIT_GROUPS_ONLY=str(i))
    try:
        r = subprocess.run([sys.executable, "-c", code, f"/tmp/g{i}.npy"], env=env, capture_output=True, text=True,
                           timeout=120)
        got = np.load(f"/tmp/g{i}.npy")
        diff = np.abs(got - ref)
        print(i, "identical" if np.array_equal(got, ref) else f"DIFFERS max {diff.max():.3e} count {(diff > 0).sum()}",
              flush=True)
    except subprocess.TimeoutExpired:
        print(i, "TIMEOUT", flush=True)
