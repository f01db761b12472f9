"""Copy-engine overlap probe: a 16 GiB D2H on a side stream, then a marker
event and a 16 GiB H2D on the default stream.  Variants add the ingredients
of run_plan(out=...) one at a time to find what serialises them."""
import torch

n = 1 << 30
host_in = torch.zeros(n, dtype=torch.complex128).pin_memory()
host_out = torch.empty(n, dtype=torch.complex128).pin_memory()
cs = torch.cuda.Stream()


def trial(name, wait_done=False, rec_copied=False, rec_stream=False, free_src=False):
    src = torch.ones(n, dtype=torch.complex128, device="cuda")
    dst = torch.empty(n, dtype=torch.complex128, device="cuda")
    torch.cuda.synchronize()
    T0 = torch.cuda.Event(enable_timing=True)
    T0.record()
    done = torch.cuda.Event()
    done.record()
    if wait_done:
        cs.wait_event(done)
    with torch.cuda.stream(cs):
        host_out.copy_(src, non_blocking=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c1.record(cs)
        if rec_copied:
            ev = torch.cuda.Event()
            ev.record(cs)
    if rec_stream:
        src.record_stream(cs)
    if free_src:
        del src
    mark = torch.cuda.Event(enable_timing=True)
    mark.record()
    dst.copy_(host_in, non_blocking=True)
    h1 = torch.cuda.Event(enable_timing=True)
    h1.record()
    torch.cuda.synchronize()
    print(f"{name:34s} marker at {T0.elapsed_time(mark):7.1f} ms, H2D done {T0.elapsed_time(h1):7.1f}, "
          f"D2H done {T0.elapsed_time(c1):7.1f}", flush=True)


trial("plain")
trial("wait_event(done)", wait_done=True)
trial("+ copied event", wait_done=True, rec_copied=True)
trial("+ record_stream", wait_done=True, rec_copied=True, rec_stream=True)
trial("+ free src", wait_done=True, rec_copied=True, rec_stream=True, free_src=True)
trial("record_stream + free only", rec_stream=True, free_src=True)

# the same trial after the executor has run once (its streams, its library)
import sys  # noqa: E402
from pathlib import Path  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2509_14098_b200.executor as ex  # noqa: E402
from paper_2509_14098_b200 import plan as planmod, run_plan  # noqa: E402

plan = planmod.load(str(Path(__file__).resolve().parent.parent / "plans" / "qft30_h30-12.json.gz"))
host_in[0] = 1.0
run_plan(plan, initial=host_in.view(1, n), out=host_out.view(1, n)).wait()
trial("after run_plan, fresh stream")
cs = list(ex._COPY_STREAMS.values())[0]
trial("after run_plan, executor copy stream")
run_plan(plan).state  # a plain run (no out=)
trial("after a plain run_plan")

# run_plan without out=, then the same download block in user code
for k in range(2):
    r = run_plan(plan, initial=host_in.view(1, n))
    T0 = torch.cuda.Event(enable_timing=True)
    T0.record()
    done = torch.cuda.Event()
    done.record()
    cs.wait_event(done)
    with torch.cuda.stream(cs):
        host_out.view(1, n).copy_(r.state.blocks, non_blocking=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c1.record(cs)
    mark = torch.cuda.Event(enable_timing=True)
    mark.record()
    torch.cuda.synchronize()
    print(f"user-side download of run_plan state: marker {T0.elapsed_time(mark):.1f} ms, D2H done {T0.elapsed_time(c1):.1f}",
          flush=True)
    r2 = run_plan(plan, initial=host_in.view(1, n), out=host_out.view(1, n))
    mark = torch.cuda.Event(enable_timing=True)
    mark.record()
    torch.cuda.synchronize()
    print(f"run_plan(out=): marker after return {r2.copied.elapsed_time(mark) if False else 0:.1f}", flush=True)
    del r, r2


def user_dl(name, t):
    torch.cuda.synchronize()
    T0 = torch.cuda.Event(enable_timing=True)
    T0.record()
    with torch.cuda.stream(cs):
        host_out.view(-1)[:t.numel()].copy_(t.reshape(-1), non_blocking=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c1.record(cs)
    mark = torch.cuda.Event(enable_timing=True)
    mark.record()
    torch.cuda.synchronize()
    print(f"{name:40s} marker {T0.elapsed_time(mark):7.1f} ms, D2H done {T0.elapsed_time(c1):7.1f}", flush=True)


r = run_plan(plan, initial=host_in.view(1, n))
user_dl("state after run with initial", r.state.blocks)
user_dl("clone of that state", r.state.blocks.clone())
del r
r = run_plan(plan)
user_dl("state after run from |0>", r.state.blocks)
del r
x = torch.empty(n, dtype=torch.complex128, device="cuda")
x.copy_(host_in, non_blocking=True)
torch.cuda.synchronize()
user_dl("tensor filled by H2D", x)
import paper_2509_14098_b200._native as nat  # noqa: E402
lib = nat.load()
nat.check(lib.svb_norm2(x.data_ptr(), 16, torch.zeros(1, dtype=torch.float64, device="cuda").data_ptr(),
                        torch.cuda.current_stream().cuda_stream), "n")
torch.cuda.synchronize()
user_dl("after a libsvb200 kernel", x)

comp = ex.compile_plan(plan, ex.prog.DeviceGeometry(d=30, g=0, h=0, rank_base=0, pad_to=4),
                       torch.device("cuda", 0), None, zero_start=False)
y = torch.zeros(n, dtype=torch.complex128, device="cuda")
y[0] = 1
torch.cuda.synchronize()
user_dl("fresh tensor before a JIT sweep", y)
nat.check(lib.svb_jit_launch_sweep(comp.kernels[0], y.data_ptr(), comp.blob.data_ptr(), comp.descs[0:1].ctypes.data,
                                   None, 0, torch.cuda.current_stream().cuda_stream), "jit")
torch.cuda.synchronize()
user_dl("after one JIT sweep on it", y)
z = torch.zeros(n, dtype=torch.complex128, device="cuda")
torch.cuda.synchronize()
user_dl("another fresh tensor after JIT", z)

r = run_plan(plan)
b = r.state.blocks
print("state tensor:", b.shape, b.stride(), b.storage_offset(), b.is_contiguous(), b.dtype, b.device,
      "base" if b._base is not None else "nobase", b.untyped_storage().nbytes(), flush=True)
print("plain tensor:", z.shape, z.stride(), z.storage_offset(), z.is_contiguous(), z.untyped_storage().nbytes(), flush=True)
import ctypes, glob  # noqa: E402,E401
cands = glob.glob(str(Path(torch.__file__).parent / "lib" / "libcudart*.so*")) + glob.glob("/usr/local/cuda/lib64/libcudart.so*")
rt = ctypes.CDLL(cands[0])
rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
torch.cuda.synchronize()
T0 = torch.cuda.Event(enable_timing=True)
T0.record()
with torch.cuda.stream(cs):
    assert rt.cudaMemcpyAsync(host_out.data_ptr(), b.data_ptr(), 16 * n, 2, cs.cuda_stream) == 0
    c1 = torch.cuda.Event(enable_timing=True)
    c1.record(cs)
mark = torch.cuda.Event(enable_timing=True)
mark.record()
torch.cuda.synchronize()
print(f"raw cudaMemcpyAsync of the state: marker {T0.elapsed_time(mark):.1f} ms, D2H done {T0.elapsed_time(c1):.1f}", flush=True)
user_dl("torch copy_ of b.view(-1)", b.view(-1))
user_dl("torch copy_ of b[0]", b[0])
user_dl("state, first half", b.view(-1)[: n // 2])
user_dl("state, second half", b.view(-1)[n // 2:])
b.mul_(1.0)
torch.cuda.synchronize()
user_dl("state after b.mul_(1.0)", b.view(-1))
del r, b
r = run_plan(plan)
torch.cuda.synchronize()
w = torch.empty(n, dtype=torch.complex128, device="cuda")
w.copy_(r.state.blocks.view(-1))
torch.cuda.synchronize()
user_dl("fresh copy of a new state", w)
user_dl("the new state again", r.state.blocks.view(-1))
print("sweep kernels:", len(ex._compile_cache), flush=True)

small = torch.zeros(8, dtype=torch.float64, device="cuda")
big = torch.ones(n, dtype=torch.complex128, device="cuda")
pin8 = torch.empty(8, dtype=torch.float64).pin_memory()
torch.cuda.synchronize()
small.cpu()
user_dl("after a pageable small .cpu()", big)
small.add_(1)
small.cpu()
small.add_(1)
user_dl("pageable .cpu() then a tiny kernel", big)
pin8.copy_(small, non_blocking=True)
torch.cuda.current_stream().synchronize()
user_dl("after a pinned non_blocking small read", big)
