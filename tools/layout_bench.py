"""Layout kernel throughput on one GPU: out-of-place storage<->basis bit
permutations (svb_bitperm: gather/scatter) and in-place bit swaps
(svb_bitswap: initial-state layouts), on 2^30 amplitudes.  Prints JSON."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_14098_b200 import _native  # noqa: E402

lib = _native.load()
n_bits = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n = 1 << n_bits
src = torch.empty(n, dtype=torch.complex128, device="cuda")
dst = torch.empty_like(src)
st = torch.cuda.current_stream().cuda_stream
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


out = {"amplitudes": n}
perms = {
    "reverse": list(range(n_bits - 1, -1, -1)),
    "rotate_low_to_high": [(k + n_bits - 5) % n_bits for k in range(n_bits)],
    "identity": list(range(n_bits)),
}
for name, perm in perms.items():
    arr, p32 = _native.i32_array(perm)
    ms = timed(lambda: _native.check(lib.svb_bitperm(src.data_ptr(), dst.data_ptr(), n_bits, p32, st), "bitperm"))
    out[f"bitperm_{name}"] = {"ms": ms, "gbs": 32 * n / ms / 1e6, "frac": 32 * n / ms / 1e6 / peak}
for name, pairs in {"swap_low3_high3": [(0, n_bits - 1), (1, n_bits - 2), (2, n_bits - 3)],
                    "swap_mid": [(8, 20), (9, 21)]}.items():
    u = np.asarray([a for a, _ in pairs], dtype=np.int32)
    w = np.asarray([b for _, b in pairs], dtype=np.int32)
    ms = timed(lambda: _native.check(lib.svb_bitswap(src.data_ptr(), n_bits, u.ctypes.data_as(_native._pi32),
                                                     w.ctypes.data_as(_native._pi32), len(pairs), st), "bitswap"))
    out[f"bitswap_{name}"] = {"ms": ms, "gbs": 32 * n / ms / 1e6, "frac": 32 * n / ms / 1e6 / peak}
print(json.dumps(out))
