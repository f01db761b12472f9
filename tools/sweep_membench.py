"""Memory-path microbenchmark: the sweep kernel with empty programs.

Each config is a tile bit set over a 2^D-amplitude state; the kernel only
loads and stores tiles, so GB/s = 32 B x 2^D / time shows how the tile
shape (contiguous run length, page spread) and grid size affect the
achievable bandwidth.
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2509_14098_b200 import _native, program as prog  # noqa: E402


def empty_desc(tile_bits, D):
    K = len(tile_bits)
    buf = prog.ProgramBuffers()
    sp = prog.SweepProgram(K=K, tin=sorted(tile_bits), items=[prog._Item(prog.OP_PHALL, ())],
                           out_map={b: (b, 0) for b in tile_bits})
    geo = prog.DeviceGeometry(d=D, g=0, h=0, rank_base=0)
    prog.emit_sweep(sp, geo, buf)
    return prog.pack(buf)


CONFIGS = {
    "contig_0-11": list(range(12)),
    "run8_0-2+21-29": list(range(3)) + list(range(21, 30)),
    "run4_0-1+20-29": list(range(2)) + list(range(20, 30)),
    "run2_0+19-29": [0] + list(range(19, 30)),
    "run1_18-29": list(range(18, 30)),
    "run1_6-11+18-23": list(range(6, 12)) + list(range(18, 24)),
    "run16_0-3+9-16": list(range(4)) + list(range(9, 17)),
    "run8_0-2+8-16": list(range(3)) + list(range(8, 17)),
    "run1_8-19": list(range(8, 20)),
    "contig_0-9": list(range(10)),
    "run8_0-2+23-29": list(range(3)) + list(range(23, 30)),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--D", type=int, default=30)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    D = a.D
    lib = _native.load()
    state = torch.zeros(1 << D, dtype=torch.complex128, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for name, bits in CONFIGS.items():
        blob, descs, _ = empty_desc(bits, D)
        dblob = torch.from_numpy(blob).cuda()
        for grid in (0, 296):
            def run():
                _native.check(lib.svb_run_sweeps(state.data_ptr(), 1, D, dblob.data_ptr(),
                                                 descs.ctypes.data, 1, None, grid, st), "sweep")
            run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3 / a.reps
            print(f"{name:22s} grid={grid:4d} K={len(bits)} {t * 1e3:8.2f} ms "
                  f"{32 * (1 << D) / t / 1e9:8.1f} GB/s", flush=True)
    dst = torch.empty_like(state)
    dst.copy_(state)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        dst.copy_(state)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / a.reps
    print(f"torch copy {32 * (1 << D) / t / 1e9:8.1f} GB/s")


main()
