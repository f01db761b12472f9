"""Event timeline of pipelined run_plan(initial=..., out=...) steps: when does
each step's upload run relative to the previous step's download?"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2509_14098_b200.executor as ex  # noqa: E402
from paper_2509_14098_b200 import plan as planmod, run_plan  # noqa: E402

import os  # noqa: E402
if os.environ.get("PROBE_NO_RECORD"):
    torch.Tensor.record_stream = lambda self, s: None
plan = planmod.load(str(ROOT / "plans" / "qft30_h30-12.json.gz"))
n = 1 << 30
host_in = torch.zeros((1, n), dtype=torch.complex128).pin_memory()
host_in[0, 0] = 1
host_out = torch.empty((1, n), dtype=torch.complex128).pin_memory()
T0 = torch.cuda.Event(enable_timing=True)
marks = []
orig = ex._load_initial


def traced(state, *a, **k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t = time.perf_counter()
    orig(state, *a, **k)
    marks.append(("h2d issue host ms", 1e3 * (time.perf_counter() - t)))
    e1.record()
    marks.append(("h2d", e0, e1))


ex._load_initial = traced


def wrap(name):
    fn = getattr(ex, name)

    def inner(*a, **k):
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn(*a, **k)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        marks.append((name, e0, e1))
        return out
    setattr(ex, name, inner)


wrap("compile_plan")
orig_state = ex._State


class State(orig_state):
    def __init__(self, *a, **k):
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        super().__init__(*a, **k)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        marks.append(("_State", e0, e1))


ex._State = State
run_plan(plan, initial=host_in, out=host_out).wait()
torch.cuda.synchronize()
T0.record()
import os as _os  # noqa: E402
ASYNC = _os.environ.get("PROBE_ASYNC") == "1"
rs = []
prev = None
for i in range(3):
    t = time.perf_counter()
    eb = torch.cuda.Event(enable_timing=True)
    eb.record()
    r = run_plan(plan, initial=host_in, out=host_out, wait=not ASYNC)
    t_call = time.perf_counter()
    if ASYNC:
        if prev is not None:
            prev.wait()
        prev = r
    marks.append((f"step {i} run_plan host ms", 1e3 * (t_call - t)))
    marks.append((f"step {i} prev.wait host ms", 1e3 * (time.perf_counter() - t_call)))
    ea = torch.cuda.Event(enable_timing=True)
    ea.record()
    marks.append((f"step {i} start", eb, eb))
    marks.append((f"step {i} after return", ea, ea))
    ec = torch.cuda.Event(enable_timing=True)
    ec.record(list(ex._COPY_STREAMS.values())[0])
    marks.append((f"step {i} copy stream tail", ec, ec))
    marks.append((f"step {i} host ms", 1e3 * (time.perf_counter() - t)))
    cs = ex._COPY_STREAMS[torch.device("cuda", 0)] if torch.device("cuda", 0) in ex._COPY_STREAMS else list(ex._COPY_STREAMS.values())[0]
    rs.append(r.copied)
    ec2 = torch.cuda.Event(enable_timing=True)
    ec2.record(list(ex._COPY_STREAMS.values())[0])
    marks.append((f"step {i} copy-stream tail (incl. this D2H)", ec2, ec2))
    del r
    ed = torch.cuda.Event(enable_timing=True)
    ed.record()
    marks.append((f"step {i} after del", ed, ed))
torch.cuda.synchronize()
for m in marks:
    if len(m) == 2:
        print(f"{m[0]}: {m[1]:.1f}")
    else:
        print(f"{m[0]}: {T0.elapsed_time(m[1]):.1f} -> {T0.elapsed_time(m[2]):.1f} ms")
print("streams: current", torch.cuda.current_stream(), "copy", list(ex._COPY_STREAMS.values()))
