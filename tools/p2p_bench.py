"""NVLink ceilings between two processes (one GPU each) over CUDA IPC:
SM push (local -> peer stores), SM pull (peer -> local loads), copy-engine
peer copy, both directions at once, and the in-place swap kernel.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2p_bench.py
"""
import ctypes
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2509_14098_b200 import _native, comm  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    me = dist.get_rank()
    peer = 1 - me
    lib = _native.load()
    n = 1 << 30  # 16 GiB of amplitudes per process
    buf, ctx = comm.symmetric_buffer(n, dev, None)
    peers = ctx.peers
    buf.fill_(1.0 + me)
    pbase = peers[peer]
    st = torch.cuda.current_stream().cuda_stream
    half = n // 2
    nbytes_half = half * 16

    def timed(fn, reps=3):
        fn()
        comm.device_barrier(None, dev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 1e3 / reps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def out(name, bytes_per_dir, t):
        if me == 0:
            print(f"{name:44s} {t * 1e3:8.2f} ms  {bytes_per_dir / t / 1e9:7.1f} GB/s per direction", flush=True)

    src = buf.data_ptr()  # my first half
    dst_remote = pbase + nbytes_half  # peer's second half
    src_remote = pbase  # peer's first half
    dst_local = buf.data_ptr() + nbytes_half
    for grid in (0,):
        t = timed(lambda: _native.check(lib.svb_copy(dst_remote, src, half, grid, st), "copy"))
        out(f"SM push 8 GiB both ways (grid {grid or 'auto'})", nbytes_half, t)
    for grid in (0,):
        t = timed(lambda: _native.check(lib.svb_copy(dst_local, src_remote, half, grid, st), "copy"))
        out(f"SM pull 8 GiB both ways (grid {grid or 'auto'})", nbytes_half, t)
    # copy engine: cudaMemcpyAsync D2D on UVA pointers
    t = timed(lambda: _ce(dst_remote, src, nbytes_half, st))
    out("CE push 8 GiB both ways", nbytes_half, t)
    # in-place swap: m = 1 on the top local bit, region = 8 GiB, pairs split in half
    lb = np.asarray([29], dtype=np.int32)
    sel_l = np.asarray([1 - me], dtype=np.uint64)
    sel_r = np.asarray([me], dtype=np.uint64)
    region = half
    first = np.asarray([0 if me == 0 else region // 2], dtype=np.int64)
    count = np.asarray([region // 2], dtype=np.int64)
    ptrs = (ctypes.c_void_p * 1)(pbase)
    for grid, block in ((0, 256), (16, 1024), (32, 1024)):
        t = timed(lambda: _native.check(lib.svb_peer_swap(buf.data_ptr(), ptrs, 1, 1, 30,
                                                          lb.ctypes.data_as(_native._pi32), 1,
                                                          sel_l.ctypes.data, sel_r.ctypes.data,
                                                          first.ctypes.data, count.ctypes.data, grid, block,
                                                          st),
                                        "swap"))
        out(f"swap kernel m=1 (grid {grid or 'auto'} x {block})", nbytes_half, t)
    # bulk (TMA-engine) swap: NVLink rate vs number of SMs
    for grid, piece, stages, ahead in ((148, 16384, 6, 4), (16, 16384, 6, 4), (16, 16384, 6, 2),
                                       (16, 16384, 6, 3), (12, 16384, 6, 3), (8, 16384, 6, 3),
                                       (16, 8192, 12, 6), (16, 8192, 12, 4), (12, 32768, 3, 1),
                                       (148, 4096, 3, 1), (148, 4096, 3, 2), (148, 8192, 2, 1)):
        t = timed(lambda: _native.check(lib.svb_peer_swap_bulk(buf.data_ptr(), ptrs, 1, 1, 30,
                                                               lb.ctypes.data_as(_native._pi32), 1,
                                                               sel_l.ctypes.data, sel_r.ctypes.data,
                                                               first.ctypes.data, count.ctypes.data,
                                                               grid, piece, stages, ahead, st),
                                        "bulk"))
        out(f"bulk swap (grid {grid}, piece {piece}, stages {stages}, ahead {ahead})", nbytes_half, t)
    # correctness: tagged data, swap on bit lb, expected value known in closed form
    idx = torch.arange(n, device=dev, dtype=torch.float64)
    for kind in ("reg", "bulk"):
        for lbit in (29, 5, 0):
            buf.real.copy_(idx)
            buf.imag.fill_(float(me))
            comm.device_barrier(None, dev)
            lbv = np.asarray([lbit], dtype=np.int32)
            args = (buf.data_ptr(), ptrs, 1, 1, 30, lbv.ctypes.data_as(_native._pi32), 1, sel_l.ctypes.data,
                    sel_r.ctypes.data, first.ctypes.data, count.ctypes.data)
            if kind == "reg":
                _native.check(lib.svb_peer_swap(*args, 0, 0, st), "swap")
            else:
                _native.check(lib.svb_peer_swap_bulk(*args, 16, 16384, 6, 3, st), "bulk")
            comm.device_barrier(None, dev)
            torch.cuda.synchronize()
            ii = torch.arange(n, device=dev, dtype=torch.int64)
            moved = ((ii >> lbit) & 1) == (1 - me)
            want_re = torch.where(moved, (ii ^ (1 << lbit)).double(), ii.double())
            want_im = torch.where(moved, torch.full_like(idx, float(peer)), torch.full_like(idx, float(me)))
            bad = int(((buf.real != want_re) | (buf.imag != want_im)).sum().item())
            t = torch.tensor([bad], device=dev)
            dist.all_reduce(t)
            if me == 0:
                print(f"check {kind} swap lbit {lbit}: {int(t.item())} wrong amplitudes", flush=True)
            del ii, moved, want_re, want_im
    dist.destroy_process_group()


_cudart = None


def _ce(dst, src, nbytes, st):
    global _cudart
    if _cudart is None:
        import glob

        cands = glob.glob(str(Path(torch.__file__).parent / "lib" / "libcudart*.so*"))
        cands += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
        _cudart = ctypes.CDLL(cands[0])
        _cudart.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                            ctypes.c_void_p]
    rc = _cudart.cudaMemcpyAsync(dst, src, nbytes, 3, st)
    assert rc == 0, rc


main()
