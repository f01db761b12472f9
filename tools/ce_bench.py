"""Copy-engine bandwidth: peer copies GPU0 <-> GPU1 (one process, two GPUs),
single and bidirectional, plus an on-device D2D copy."""
import torch


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream(0))
    for _ in range(reps):
        fn()
    e1.record(torch.cuda.current_stream(0))
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    return e0.elapsed_time(e1) / 1e3 / reps


n = (1 << 30) // 16  # 1 GiB of complex128
a0 = torch.ones(n, dtype=torch.complex128, device="cuda:0")
b0 = torch.empty_like(a0)
a1 = torch.ones(n, dtype=torch.complex128, device="cuda:1")
b1 = torch.empty_like(a1)
print("peer access 0->1:", torch.cuda.can_device_access_peer(0, 1))
t = timed(lambda: b1.copy_(a0, non_blocking=True))
print(f"CE peer copy 0->1 (1 GiB): {(1 << 30) / t / 1e9:.1f} GB/s")
s1 = torch.cuda.Stream(device=1)


def bidir():
    b1.copy_(a0, non_blocking=True)
    with torch.cuda.stream(s1):
        b0.copy_(a1, non_blocking=True)


t = timed(bidir)
print(f"CE bidirectional (1 GiB each way): {(1 << 30) / t / 1e9:.1f} GB/s per direction")
t = timed(lambda: b0.copy_(a0, non_blocking=True))
print(f"on-device D2D copy (1 GiB): {2 * (1 << 30) / t / 1e9:.1f} GB/s (read+write)")
# strided (2D) peer copy: 64 runs of 16 MiB with a 32 MiB pitch
src = a0.view(64, -1)[:, : n // 128]
dst = b1.view(64, -1)[:, : n // 128]
t = timed(lambda: dst.copy_(src, non_blocking=True))
print(f"CE 2D peer copy (64 x 8 MiB runs): {(1 << 29) / t / 1e9:.1f} GB/s")
