"""Compare the JIT and interpreter sweep paths sweep-by-sweep on golden cases."""
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_14098_b200 import _native, executor, jit, plan as planmod, program as prog  # noqa: E402

docs = json.load(gzip.open(ROOT / "tests/golden/grid.json.gz", "rt"))
if len(sys.argv) > 1:  # plans/<name>.json.gz instead of the grid
    docs = [{"name": n, "plan": json.loads(planmod.to_json(planmod.load(str(ROOT / "plans" / f"{n}.json.gz"))))}
            for n in sys.argv[1:]]
lib = _native.load()
bad = 0
for doc in docs:
    plan = planmod.from_json(json.dumps(doc["plan"]))
    if plan.d < 8:
        continue
    L = plan.d - plan.g
    geo = prog.DeviceGeometry(d=plan.d, g=plan.g, h=plan.g, rank_base=0, pad_to=4)
    buf4 = prog.plan_device(plan, geo, rb=4).buf  # interpreter program
    buf = prog.plan_device(plan, geo, rb=3).buf  # JIT program (same sweeps)
    blob4, descs4, _ = prog.pack(buf4)
    dblob4 = torch.from_numpy(blob4).cuda()
    blob, descs, _ = prog.pack(buf)
    dblob = torch.from_numpy(blob).cuda()
    names, cubins = jit.build_kernels(buf)
    kern = [jit.load_kernel(n, c, 0) for n, c in zip(names, cubins)]
    rng = np.random.default_rng(0)
    n = 1 << geo.D
    v = rng.normal(size=n) + 1j * rng.normal(size=n)
    v /= np.linalg.norm(v)
    for i in range(len(descs)):
        a = torch.from_numpy(v.copy()).cuda()
        b = torch.from_numpy(v.copy()).cuda()
        st = torch.cuda.current_stream().cuda_stream
        _native.check(lib.svb_run_sweeps(a.data_ptr(), 1 << (geo.D - L), L, dblob4.data_ptr(),
                                         descs4[i:i + 1].ctypes.data, 1, None, 0, st), "interp")
        _native.check(lib.svb_jit_launch_sweep(kern[i], b.data_ptr(), dblob.data_ptr(),
                                               descs[i:i + 1].ctypes.data, None, 0, st), "jit")
        torch.cuda.synchronize()
        err = (a - b).abs().max().item()
        if err > 1e-12:
            bad += 1
            d = buf.descs[i]
            ops = buf.ops[d["op_begin"]: d["op_begin"] + d["op_count"]]
            print("MISMATCH", doc["name"], "sweep", i, "err", err, "K", d["K"], "D", d["D"],
                  "kinds", [o["kind"] for o in ops])
            if bad == 1:
                open(ROOT / "gpurun_out" / "bad_kernel.cu", "w").write(
                    jit.kernel_source("bad", d, ops, buf.coef))
                print([dict((k, o[k]) for k in o) for o in ops][:6])
            break
    if bad >= 6:
        break
print("done, mismatching cases:", bad)
