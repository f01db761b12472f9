"""A/B one sweep: its one-group and two-group kernels on the same random
state (fresh copies), compared bit for bit; prints where they differ."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_14098_b200 import _native, jit, plan as planmod, program as prog  # noqa: E402

name, di = sys.argv[1], int(sys.argv[2])
plan = planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))
geo = prog.DeviceGeometry(d=plan.d, g=plan.g, h=plan.g, rank_base=0, pad_to=4)
dp = prog.plan_device(plan, geo, rb=4, free_start=True)
blob, descs, _ = prog.pack(dp.buf)
dblob = torch.from_numpy(blob).cuda()
d = dp.buf.descs[di]
ops = dp.buf.ops[d["op_begin"]: d["op_begin"] + d["op_count"]]
lib = _native.load()
n = 1 << geo.D
gen = torch.Generator(device="cuda").manual_seed(1)
x0 = torch.randn(n, dtype=torch.complex128, device="cuda", generator=gen)
outs = {}
for tag, fn, groups in (("1g", jit.kernel_source, 0), ("2g", jit.kernel_source_2g, 2)):
    kname = f"ab_{tag}_{di}"
    src = fn(kname, d, ops, dp.buf.coef, 0, None)
    cub = jit._compile(src, kname)
    k = jit.load_kernel(kname, cub, 0)
    desc = descs[di:di + 1].copy()
    desc[0]["groups"] = groups
    x = x0.clone()
    norms = torch.zeros(64, dtype=torch.float64, device="cuda")
    _native.check(lib.svb_jit_launch_sweep(k, x.data_ptr(), dblob.data_ptr(), desc.ctypes.data, norms.data_ptr(), 0,
                                           torch.cuda.current_stream().cuda_stream), "launch")
    torch.cuda.synchronize()
    outs[tag] = x
    print(tag, "norm", norms[int(d["norm_slot"])].item() if int(d["norm_slot"]) >= 0 else None, flush=True)
diff = (outs["1g"] != outs["2g"])
bad = torch.nonzero(diff).flatten()
print("differing amplitudes:", bad.numel(), "of", n)
if bad.numel():
    tin = [int(b) for b in d["tin"][:d["K"]]]
    fbits = [b for b in range(geo.D) if b not in tin]
    idx = bad[:2000].cpu().numpy()
    tiles = np.zeros_like(idx)
    for i, b in enumerate(fbits):
        tiles |= ((idx >> b) & 1) << i
    u, c = np.unique(tiles, return_counts=True)
    print("tiles with differences:", len(u), "first", u[:20], "counts", c[:20])
    print("grid 148 -> CTA", (u[:20] % 148), "k", (u[:20] // 148))
