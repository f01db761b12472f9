"""Interference between a fused sweep and the peer swap kernel (2 processes,
one GPU each): each alone, then both at once on separate streams.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/contend.py
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

from paper_2509_14098_b200 import _native, comm, executor, jit, plan as planmod, program as prog  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    me = dist.get_rank()
    lib = _native.load()
    # the 2-GPU QFT-31 program with overlap planning: chunked sweeps are
    # compiled for part launches with the overlap register cap
    plan = planmod.load(str(ROOT / "plans" / "qft31_h30-12.json.gz"))
    geo = prog.DeviceGeometry(d=plan.d, g=plan.g, h=0, rank_base=me, pad_to=4)
    dp = prog.plan_device(plan, geo, rb=4, overlap_bits=3)
    blob, descs, _ = prog.pack(dp.buf)
    dblob = torch.from_numpy(blob).to(dev)
    names, cubins = jit.build_kernels(dp.buf)
    kern = [jit.load_kernel(n, c, local) for n, c in zip(names, cubins)]

    class Comp:
        pass

    comp = Comp()
    comp.descs, comp.blob, comp.kernels = descs, dblob, kern
    n = 1 << 30
    buf, ctx = comm.symmetric_buffer(n, dev, None)
    buf.zero_()
    peer = 1 - me
    s_sweep = torch.cuda.Stream()
    s_swap = torch.cuda.Stream()
    lb = np.asarray([29], dtype=np.int32)
    sel_l = np.asarray([1 - me], dtype=np.uint64)
    sel_r = np.asarray([me], dtype=np.uint64)
    region = n // 2
    first = np.asarray([0 if me == 0 else region // 2], dtype=np.int64)
    count = np.asarray([region // 2], dtype=np.int64)
    ptrs = (ctypes.c_void_p * 1)(ctx.peers[peer])

    class St:
        pass

    stt = St()
    stt.buf = buf
    which = [2]

    def sweep(_):
        i = which[0]
        cb = dp.buf.descs[i].get("cbits")
        if cb:
            with torch.cuda.stream(s_sweep):
                for c in range(1 << len(cb)):
                    executor._launch_part(comp, i, stt, None, 0, s_sweep.cuda_stream, cb, c)
        else:
            _native.check(lib.svb_jit_launch_sweep(kern[i], buf.data_ptr(), dblob.data_ptr(),
                                                   descs[i:i + 1].ctypes.data, None, 0, s_sweep.cuda_stream),
                          "sw")

    def swap(grid, piece, stages, ahead):
        _native.check(lib.svb_peer_swap_bulk(buf.data_ptr(), ptrs, 1, 1, 30, lb.ctypes.data_as(_native._pi32), 1,
                                             sel_l.ctypes.data, sel_r.ctypes.data, first.ctypes.data,
                                             count.ctypes.data, grid, piece, stages, ahead, s_swap.cuda_stream),
                      "swap")

    def run(do_sweep, cfg):
        torch.cuda.synchronize()
        comm.device_barrier(None, dev)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(s_sweep)
        ev[2].record(s_swap)
        if do_sweep:
            sweep(2)
        if cfg:
            swap(*cfg)
        ev[1].record(s_sweep)
        ev[3].record(s_swap)
        torch.cuda.synchronize()
        t = torch.tensor([ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    for i in (1, 2, 3, 4):
        which[0] = i
        for _ in range(2):
            run(True, None)
        ts = run(True, None)[0]
        if me == 0:
            print(f"sweep {i} (cbits {dp.buf.descs[i].get('cbits')}) alone: {ts:.2f} ms", flush=True)
        for cfg in ((148, 4096, 3, 1), (148, 16384, 6, 4)):
            run(False, cfg)
            tx = run(False, cfg)[1]
            both = run(True, cfg)
            if me == 0:
                print(f"  swap {cfg}: alone {tx:.2f} ms; concurrent: sweep {both[0]:.2f} ms, swap {both[1]:.2f} ms",
                      flush=True)
    dist.destroy_process_group()


main()
