"""HBM bandwidth by access mode on one GPU: write-only, read+write, read-only.

The sparse-start sweeps are write-dominated (the last one writes the whole
state and reads a quarter), so their roofline is the write-mode bandwidth,
not the copy bandwidth in MEASURED_PEAKS.json.  Prints one JSON line."""
import json

import torch


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best / 1e3


n = 1 << 30  # complex128 amplitudes: 16 GiB
x = torch.empty(n, dtype=torch.complex128, device="cuda")
y = torch.empty(n, dtype=torch.complex128, device="cuda")
B = 16 * n
out = {
    "write_only_fill_gbs": B / timed(lambda: x.fill_(0)) / 1e9,
    "copy_rw_gbs": 2 * B / timed(lambda: y.copy_(x)) / 1e9,
    "read_only_sum_gbs": B / timed(lambda: torch.view_as_real(x).sum()) / 1e9,
}
xs = x[: n // 4]
out["read_quarter_write_all_gbs"] = (B // 4 + B) / timed(lambda: (y.view(4, -1).copy_(xs.unsqueeze(0).expand(4, -1)))) / 1e9
print(json.dumps(out))
