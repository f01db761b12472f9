"""Where the end-to-end step time goes on one GPU: PCIe copies of a 16 GiB
state (H2D, D2H, both directions at once) and run_plan with and without a
host initial state."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2509_14098_b200 import plan as planmod, run_plan  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


plan = planmod.load(str(ROOT / "plans" / "qft30_h30-12.json.gz"))
n = 1 << 30
host_in = torch.zeros(n, dtype=torch.complex128).pin_memory()
host_in[0] = 1
host_out = torch.empty(n, dtype=torch.complex128).pin_memory()
dev = torch.empty(n, dtype=torch.complex128, device="cuda")
dev2 = torch.empty(n, dtype=torch.complex128, device="cuda")
s2 = torch.cuda.Stream()
print(f"H2D 16 GiB: {timed(lambda: dev.copy_(host_in, non_blocking=True)):.1f} ms", flush=True)
print(f"D2H 16 GiB: {timed(lambda: host_out.copy_(dev, non_blocking=True)):.1f} ms", flush=True)


def duplex():
    dev.copy_(host_in, non_blocking=True)
    with torch.cuda.stream(s2):
        host_out.copy_(dev2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


print(f"H2D + D2H concurrently: {timed(duplex):.1f} ms", flush=True)
del dev, dev2
blocks_in = host_in.view(1, n)


def with_initial():
    r = run_plan(plan, initial=blocks_in)
    host_out.view(1, n).copy_(r.state.blocks, non_blocking=True)
    torch.cuda.synchronize()


def from_zero():
    r = run_plan(plan)
    torch.cuda.synchronize()
    del r


print(f"run_plan(initial=host) + D2H: {timed(with_initial):.1f} ms", flush=True)
print(f"run_plan from |0> (device only): {timed(from_zero):.1f} ms", flush=True)
r = run_plan(plan, initial=blocks_in)
print("stats", {k: round(v * 1e3, 2) for k, v in vars(r.stats).items() if k.endswith("seconds")}, flush=True)


def pipelined(steps=5):
    rs = []
    for _ in range(steps):
        r = run_plan(plan, initial=blocks_in, out=host_out.view(1, n))
        rs.append(r.copied)
        del r
    torch.cuda.synchronize()


t0 = time.perf_counter()
pipelined()
print(f"pipelined run_plan(initial, out=) x5: {(time.perf_counter() - t0) / 5 * 1e3:.1f} ms/step", flush=True)
# host-side timeline of one pipelined step
import paper_2509_14098_b200.executor as ex  # noqa: E402
for i in range(3):
    t0 = time.perf_counter()
    r = run_plan(plan, initial=blocks_in, out=host_out.view(1, n))
    t1 = time.perf_counter()
    ok = r.copied.query()
    print(f"step {i}: run_plan returned after {1e3 * (t1 - t0):.1f} ms; copy done at return: {ok}", flush=True)
    del r
torch.cuda.synchronize()
