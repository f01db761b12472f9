"""NVLink point-to-point bandwidth between rank pairs via NCCL send/recv
(torchrun, 2+ ranks): the ceiling for the remap's data movement."""
import os
import sys
import time

import torch
import torch.distributed as dist


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    me, world = dist.get_rank(), dist.get_world_size()
    peer = me ^ 1
    for mb in (64, 256, 1024):
        n = mb << 20
        a = torch.ones(n // 8, dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        for _ in range(3):
            ops = [dist.P2POp(dist.isend, a, peer), dist.P2POp(dist.irecv, b, peer)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        torch.cuda.synchronize()
        dist.barrier()
        reps = max(4, 4096 // mb)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ops = [dist.P2POp(dist.isend, a, peer), dist.P2POp(dist.irecv, b, peer)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / reps
        if me == 0:
            print(f"sendrecv {mb:5d} MiB: {n / t / 1e9:7.1f} GB/s per direction "
                  f"(NCCL_P2P_NVL_CHUNKSIZE={os.environ.get('NCCL_P2P_NVL_CHUNKSIZE')}, "
                  f"NCCL_MAX_NCHANNELS={os.environ.get('NCCL_MAX_NCHANNELS')})", flush=True)
    dist.destroy_process_group()


main()
