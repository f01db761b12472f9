"""Single-GPU check of sweep part launches: each sweep of a plan is run whole
and as 2^k parts over chunk bits outside its tile; results must match."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_14098_b200 import _native, executor, jit, plan as planmod, program as prog  # noqa: E402


def main(names):
    lib = _native.load()
    bad = 0
    for name in names:
        plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
        geo = prog.DeviceGeometry(d=plan.d, g=plan.g, h=plan.g, rank_base=0, pad_to=4)
        ref = prog.plan_device(plan, geo, rb=4)  # same sweeps, no chunk bits
        rblob, rdescs, _ = prog.pack(ref.buf)
        drblob = torch.from_numpy(rblob).cuda()
        rnames, rcubins = jit.build_kernels(ref.buf)
        rkern = [jit.load_kernel(n, c, 0) for n, c in zip(rnames, rcubins)]
        dp = prog.plan_device(plan, geo, rb=4)
        L = geo.L
        for d in dp.buf.descs:  # chunk bits: the two highest local bits outside the tile
            free = [b for b in range(L - 1, -1, -1) if b not in d["tin"][:d["K"]]]
            d["cbits"] = sorted(free[:2])
        blob, descs, _ = prog.pack(dp.buf)
        dblob = torch.from_numpy(blob).cuda()
        names_, cubins = jit.build_kernels(dp.buf)

        class C:  # the bits of _Compiled that _launch_part needs
            pass

        comp = C()
        comp.descs, comp.blob = descs, dblob
        comp.kernels = [jit.load_kernel(n, c, 0) for n, c in zip(names_, cubins)]
        rng = np.random.default_rng(1)
        n = 1 << geo.D
        v = rng.normal(size=n) + 1j * rng.normal(size=n)
        v /= np.linalg.norm(v)
        st = torch.cuda.current_stream().cuda_stream
        for i in range(min(len(descs), 6)):
            a = torch.from_numpy(v.copy()).cuda()
            b = torch.from_numpy(v.copy()).cuda()
            cb = dp.buf.descs[i]["cbits"]

            class S:
                pass

            sa = S()
            sa.buf = a
            _native.check(lib.svb_jit_launch_sweep(rkern[i], a.data_ptr(), drblob.data_ptr(),
                                                   rdescs[i:i + 1].ctypes.data, None, 0, st), "whole")
            sb = S()
            sb.buf = b
            for c in range(1 << len(cb)):
                executor._launch_part(comp, i, sb, None, 0, st, cb, c)
            torch.cuda.synchronize()
            err = (a - b).abs().max().item()
            print(name, "sweep", i, "cbits", cb, "err", err, flush=True)
            bad += err > 1e-12
    print("part_check mismatches:", bad)


main(sys.argv[1:] or ["qft20_h18-12", "qv20_h18-12", "qft24_h22-12"])
