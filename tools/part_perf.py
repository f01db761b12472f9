"""Timing of sweep part launches on one GPU: every sweep of a plan whole and
as 2^k parts over two chunk bits (the highest local bits outside its tile),
each part alone and all parts back to back."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2509_14098_b200 import _native, executor, jit, plan as planmod, program as prog  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main(name, nbits):
    lib = _native.load()
    plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
    geo = prog.DeviceGeometry(d=plan.d, g=plan.g, h=plan.g, rank_base=0, pad_to=4)
    dp = prog.plan_device(plan, geo, rb=4)
    whole_blob, whole_descs, _ = prog.pack(dp.buf)
    wn, wc = jit.build_kernels(dp.buf)
    wk = [jit.load_kernel(n, c, 0) for n, c in zip(wn, wc)]
    L = geo.L
    for d in dp.buf.descs:
        free = [b for b in range(L - 1, -1, -1) if b not in d["tin"][:d["K"]]]
        d["cbits"] = sorted(free[:nbits])
    blob, descs, _ = prog.pack(dp.buf)
    pn, pc = jit.build_kernels(dp.buf)

    class C:
        pass

    comp = C()
    comp.descs, comp.blob = descs, torch.from_numpy(blob).cuda()
    comp.kernels = [jit.load_kernel(n, c, 0) for n, c in zip(pn, pc)]
    dwb = torch.from_numpy(whole_blob).cuda()
    st = torch.cuda.current_stream().cuda_stream

    class S:
        pass

    s = S()
    s.buf = torch.zeros(1 << geo.D, dtype=torch.complex128, device="cuda")
    for i in range(len(descs)):
        cb = dp.buf.descs[i]["cbits"]
        tw = timed(lambda: _native.check(lib.svb_jit_launch_sweep(wk[i], s.buf.data_ptr(), dwb.data_ptr(),
                                                                   whole_descs[i:i + 1].ctypes.data, None, 0,
                                                                   st), "whole"))
        tp = timed(lambda: [executor._launch_part(comp, i, s, None, 0, st, cb, c) for c in range(1 << nbits)])
        t0 = timed(lambda: executor._launch_part(comp, i, s, None, 0, st, cb, 0))
        print(f"{name} sweep {i} K={descs[i]['K']} cbits {cb}: whole {tw:.2f} ms, "
              f"{1 << nbits} parts {tp:.2f} ms, one part {t0:.2f} ms", flush=True)


main(sys.argv[1] if len(sys.argv) > 1 else "qft30_h30-12", int(sys.argv[2]) if len(sys.argv) > 2 else 2)
