#!/usr/bin/env python
"""Benchmark: circuit time and HBM GB/s of the B200 executor vs the host-CPU reference.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload qft|qv|NAME]

One "step" = one full ``run_plan`` of the workload's plan (Alloc from |0..0>,
every ApplyFused sweep, every remap, norm check).  Plans are the reference
partitioner's output, generated once by tests/golden/make_golden.py and
read from plans/ (the partitioner runs unchanged on the host; its time is
reported separately in plans/plans.json).

Workloads (BASELINE.json configs): at N=1 the 34-qubit configs do not fit one
B200 (256 GiB of complex128), so the single-GPU line is cfg2, QFT-30 with
hierarchy [30, 12].  For N > 1 the default is weak scaling: QFT-(30+log2 N)
with [30, 12], 2^30 amplitudes per GPU and one inter-GPU remap.
``--workload qv`` runs QV-30 (N=1) / QV-34 [34-log2 N, 12] and
``--workload qft34`` QFT-34 [34-log2 N, 12] (N = 2, 4, 8: strong scaling);
``--workload qaoa`` QAOA-35 [32, 12] (N = 4, 8) and ``--workload sup`` SUP-36 [33, 12] (N = 8).

value   = algorithmic HBM bytes of all partition sweeps (32 B x 2^L per
          ApplyFused per rank) / device time of the step,
          summed over ranks; ms_per_step is the circuit time.
e2e     = the same bytes / time of run_plan(plan, initial=<pinned host
          rank blocks of this process>) plus the device->host copy of the
          final blocks (host<->device bytes counted for the whole job).
roofline= the fused sweep kernel (k_sweep): its algorithmic bytes / its
          CUDA-event time inside the timed steps, against the measured HBM
          copy bandwidth in MEASURED_PEAKS.json.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "circuit time & HBM GB/s, 34q QFT/QV at 1/2/4/8 B200 vs host-CPU reference"
UNIT = "GB/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
E2E_HOST_BYTES = 48 << 30  # pinned host buffers per process (in and out each)
TRAFFIC_REV = "r02c"  # profiles/traffic.json entries measured on the current sweep code
E2E_PIPELINE = os.environ.get("SVB200_E2E_PIPELINE", "1") != "0"  # two circuits in flight
PIPELINE = os.environ.get("SVB200_BENCH_PIPELINE", "1") != "0"  # timed loop: two circuits in flight when they fit


def workload_name(kind: str, n: int) -> tuple[str, str]:
    lg = n.bit_length() - 1
    if kind == "qft":
        return f"qft{30 + lg}_h30-12", "weak"
    if kind == "qv":
        return ("qv30_h30-12", "strong") if n == 1 else (f"qv34_h{34 - lg}-12", "strong")
    if kind == "qft34":
        if n == 1:
            raise SystemExit("qft34 needs 2+ GPUs: 2^34 complex128 amplitudes are 256 GiB")
        return f"qft34_h{34 - lg}-12", "strong"
    if kind == "qaoa":  # BASELINE cfg4: QAOA-35, 8 ranks of 2^32 amplitudes (64 GiB)
        if n < 4:
            raise SystemExit("qaoa (35 qubits, 512 GiB) needs 4+ GPUs")
        return "qaoa35_h32-12", "strong"
    if kind == "sup":  # BASELINE cfg5: SUP-36, 8 ranks of 2^33 amplitudes (128 GiB)
        if n < 8:
            raise SystemExit("sup (36 qubits, 1 TiB) needs 8 GPUs")
        return "sup36_h33-12", "strong"
    return kind, "weak"


def load_plan(name: str):
    from paper_2509_14098_b200 import plan as planmod

    return planmod.load(str(ROOT / "plans" / f"{name}.json.gz"))


def plan_bytes(plan) -> int:
    """Algorithmic HBM bytes of all ApplyFused sweeps, whole job."""
    fused = sum(1 for t in plan.tasks if t.kind == "ApplyFused")
    return fused * 32 * (1 << plan.d)


FP64_PEAK_TFS = 33.2  # DFMA, 16 warps/SM, measured on B200 (profiles/r01_fp64_dmma_vs_dfma.txt)


def sass_fp64_flops_per_tile(cubin: bytes) -> int:
    """FP64 flops one thread issues per tile of a generated sweep kernel:
    the kernels are straight-line per tile, so the static SASS count of
    DFMA (2 flops), DMUL and DADD (1 each) is the executed count (the
    per-kernel prologue and the norm epilogue are a few instructions)."""
    import re
    import tempfile

    with tempfile.NamedTemporaryFile(suffix=".cubin") as fh:
        fh.write(cubin)
        fh.flush()
        sass = subprocess.run(["cuobjdump", "-sass", fh.name], capture_output=True, text=True).stdout
    n_fma = len(re.findall(r"\bDFMA\b", sass))
    n_other = len(re.findall(r"\bD(?:MUL|ADD)\b", sass))
    return 2 * n_fma + n_other


def fp64_all_sweeps(plan_, prof: dict, compute_s_per_step: float, steps: int):
    """Executed FP64 flops of every sweep of one circuit / its sweep time."""
    from paper_2509_14098_b200 import executor, jit as jitmod

    comp = None
    for _, (pl, c) in executor._compile_cache.items():
        if pl is plan_:
            comp = c
    if comp is None or not comp.kernel_keys:
        return None
    total = 0
    for di in range(len(comp.kernel_keys)):
        if comp.kernel_keys[di] is None:  # merged into the sweep before it (no kernel)
            continue
        cub = jitmod._cached(comp.kernel_keys[di])
        if cub is None:
            return None
        d = comp.descs[di]
        K, D, rb = int(d["K"]), int(d["D"]), int(d["rb"])
        total += sass_fp64_flops_per_tile(cub) * (1 << (K - rb)) * (1 << (D - K))
    achieved = total / compute_s_per_step / 1e12
    return {"flops_per_step": total, "achieved": achieved, "frac": achieved / FP64_PEAK_TFS}


def fp64_roofline(plan_, di: int, launch_ms: float):
    """Executed FP64 TF/s of sweep di of the plan's compiled program."""
    from paper_2509_14098_b200 import executor, jit as jitmod

    comp = None
    for _, (pl, c) in executor._compile_cache.items():
        if pl is plan_:
            comp = c
    if comp is None or not comp.kernel_keys:
        return None
    cub = jitmod._cached(comp.kernel_keys[di])
    if cub is None:
        return None
    d = comp.descs[di]
    K, D, rb = int(d["K"]), int(d["D"]), int(d["rb"])
    per_thread = sass_fp64_flops_per_tile(cub)
    flops = per_thread * (1 << (K - rb)) * (1 << (D - K))
    achieved = flops / (launch_ms / 1e3) / 1e12
    return {"bound": "fp64", "achieved": achieved, "peak": FP64_PEAK_TFS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFS, "flops_per_launch": flops,
            "flops_note": "static SASS count of DFMA (x2), DMUL, DADD per thread per tile x threads x tiles",
            "peak_source": "measured DFMA throughput, 16 warps/SM (profiles/r01_fp64_dmma_vs_dfma.txt)"}


def peak_hbm() -> tuple[float, str]:
    try:
        return float(json.loads(PEAKS.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.out = ROOT / "gpurun_out" / f"clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.out.parent.mkdir(exist_ok=True)
            self.fh = open(self.out, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        # nvidia-smi takes a moment to start: begin the timed region only once
        # it is sampling, so its samples cover the (short) timed region
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < 3.0:
            try:
                if self.out.stat().st_size > 0:
                    break
            except OSError:
                pass
            time.sleep(0.02)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.out.exists():
            return None
        rows = []
        for line in self.out.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU reference arm
# ---------------------------------------------------------------------------

CPU_SAMPLE_PLAN = os.environ.get("SVB200_REF_SAMPLE", "qft22_h22-12")  # same family and [d, 12] hierarchy, bounded CPU time


def cpu_reference_step(plan, backend: str) -> float:
    from oracle import oracle as orc

    t0 = time.perf_counter()
    orc.run_plan(plan, backend=backend, check_norm=True)
    return time.perf_counter() - t0


def cpu_backend() -> tuple[str, str]:
    ref = ROOT / "oracle" / "_ref"
    if any(ref.glob("_core*.so")):
        return "ref", "reference"
    return "c", "port"


def cpu_baseline_line(min_seconds: float = 10.0, sample: str = CPU_SAMPLE_PLAN) -> dict:
    """The reference's CPU path on a bounded sample: full runs of the sample
    plan repeated until at least min_seconds of CPU work; value from the mean."""
    plan = load_plan(sample)
    backend, kind = cpu_backend()
    times = []
    while sum(times) < min_seconds:
        times.append(cpu_reference_step(plan, backend))
    t = sum(times) / len(times)
    return {"value": plan_bytes(plan) / t / 1e9, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{sample}: full plan of the same family/hierarchy, reference run_plan "
                      f"semantics with {'the reference _core.pyx kernels' if kind == 'reference' else 'the C port'}"
                      f", {plan.d} qubits, mean of {len(times)} runs ({t:.2f} s each, {sum(times):.1f} s total), "
                      f"host cores {os.cpu_count()}, 1 used",
            "seconds": t}


# the reference arm keeps a run within a few minutes: with many steps each
# step samples a smaller circuit of the same family and hierarchy
REF_BUDGET_S = float(os.environ.get("SVB200_REF_BUDGET_S", "240"))
REF_STEP_S = {"qft22_h22-12": 5.3, "qft20_h18-12": 1.8}  # one circuit per core, 16-core GPU boxes


def ref_sample(steps: int, warmup: int) -> str:
    if "SVB200_REF_SAMPLE" in os.environ:
        return CPU_SAMPLE_PLAN
    for name in ("qft22_h22-12", "qft20_h18-12"):
        if (steps + warmup) * REF_STEP_S[name] <= REF_BUDGET_S:
            return name
    return "qft20_h18-12"


def _ref_worker(sample: str, backend: str, n_warm: int, n_steps: int, barrier, out) -> None:
    """One host core: warm-up circuits, then (after every worker is warm)
    n_steps timed circuits of the sample plan; reports their wall time."""
    plan = load_plan(sample)
    for _ in range(n_warm):
        cpu_reference_step(plan, backend)
    barrier.wait()
    t0 = time.perf_counter()
    for _ in range(n_steps):
        cpu_reference_step(plan, backend)
    out.put(time.perf_counter() - t0)


def run_reference_arm(args) -> None:
    """The reference's CPU path with all the host cores it can use: the
    reference is single-threaded (no prange in _core.pyx), so every core
    runs its own copy of the sample circuit in a separate process; a step
    is one circuit on every core, and the value is the whole host's
    throughput (cores x algorithmic bytes / step time)."""
    import multiprocessing as mp

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # only rank 0 runs the CPU baseline under torchrun
    sample = ref_sample(args.steps, args.warmup)
    plan = load_plan(sample)
    backend, kind = cpu_backend()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    cores = int(os.environ.get("SVB200_REF_CORES", cores))
    ctx = mp.get_context("fork")  # this process never touched CUDA
    barrier, out = ctx.Barrier(cores), ctx.Queue()
    procs = [ctx.Process(target=_ref_worker, args=(sample, backend, args.warmup, args.steps, barrier, out))
             for _ in range(cores)]
    for p in procs:
        p.start()
    spans = [out.get() for _ in procs]
    for p in procs:
        p.join()
    total = max(spans)  # the host finishes when its slowest core does
    val = cores * plan_bytes(plan) * args.steps / total / 1e9
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": workload_name(args.workload, max(args.gpus, 1))[0],
                   "sample": f"{sample}: the same QFT family and [d, 12] hierarchy at "
                             f"{plan.d} qubits (the full workload takes ~70 min per run on one core; "
                             f"QFT-20 instead of QFT-22 when {args.steps} steps would exceed ~{REF_BUDGET_S:.0f} s); "
                             "value = algorithmic bytes / time, size-normalised like the GPU arm",
                   "note": "reference run_plan semantics with the reference's compiled _core.pyx "
                           f"kernels, which are single-threaded: {cores} independent copies, one per "
                           "host core, each step one circuit on every core"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{sample} full plan per core per step ({cores} processes), "
                                   f"per-core circuit {1e3 * total / args.steps:.0f} ms"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="qft")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sub-steps", type=int, default=6, help="steps of the N=1 sub-measurements (0: none)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = world
    name, scaling = workload_name(args.workload, n)
    plan = load_plan(name)

    from paper_2509_14098_b200 import executor, run_plan

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def in_flight(plan_) -> int:
        """2 when two copies of this process's state fit in 80% of the device
        memory (QFT-34 on 4 GPUs: 2 x 64 GiB of 178 GiB)."""
        state_bytes = 16 * ((1 << plan_.g) // world) << (plan_.d - plan_.g)
        total = torch.cuda.get_device_properties(local).total_memory
        return 2 if PIPELINE and 2 * state_bytes <= 0.8 * total else 1

    def warm(plan_, n):
        """Untimed runs in the timed loop's pattern (so the second in-flight
        state buffer exists before the clock starts).  Otherwise each result
        is dropped before the next run: its state buffer returns to the pool
        (at 34 qubits on 2 GPUs one state is 128 GiB of the 180)."""
        two = in_flight(plan_) == 2
        prev = None
        for _ in range(n):
            r = run_plan(plan_, wait=not two)
            if prev is not None:
                prev.wait()
            prev = r if two else None
            del r
        if prev is not None:
            prev.wait()
        del prev
        torch.cuda.synchronize()

    warm(plan, args.warmup)
    barrier()

    def timed(plan_, steps, clk_=None):
        """K full circuits, device-timed with CUDA events (max over ranks);
        every sweep launch is bracketed by events on its stream as well."""
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        acc = {"compute_s": 0.0, "launches": 0, "sweeps": 0, "sweep_bytes": 0, "prof": {}}
        executor.PROFILE_SWEEPS = True

        def collect(r):
            r.wait()  # event timings and the drift check of that circuit
            acc["compute_s"] += r.stats.compute_seconds + r.stats.layout_seconds
            acc["launches"] += r.stats.kernel_launches
            acc["sweeps"] += r.stats.sweeps
            acc["sweep_bytes"] += r.stats.sweep_bytes
            for di, lst in r.stats.sweep_profile.items():
                acc["prof"].setdefault(di, []).extend(lst)
            acc["stats"] = r.stats

        inflight = in_flight(plan_)
        barrier()
        start.record()
        prev = None
        for _ in range(steps):
            # with two circuits in flight the host enqueues circuit i+1 while
            # the GPU runs circuit i (every circuit is still computed and
            # drift-checked in full)
            r = run_plan(plan_, wait=inflight == 1)
            if prev is not None:
                collect(prev)
            prev = r
            if inflight == 1:
                collect(r)
                prev = None
            del r
        if prev is not None:
            collect(prev)
        del prev
        stop.record()
        barrier()
        executor.PROFILE_SWEEPS = False
        acc["elapsed"] = max_over_ranks(start.elapsed_time(stop) / 1e3)
        acc["compute_s"] = max_over_ranks(acc["compute_s"])
        return acc

    with ClockSampler(local) as clk:
        acc = timed(plan, args.steps)
    elapsed, compute_s, launches, stats = acc["elapsed"], acc["compute_s"], acc["launches"], acc["stats"]

    total_bytes = plan_bytes(plan)
    value = total_bytes * args.steps / elapsed / 1e9
    peak, peak_kind = peak_hbm()
    rows = (1 << plan.g) // world
    fused = sum(1 for t in plan.tasks if t.kind == "ApplyFused")
    sweeps = int(max_over_ranks(float(acc["sweeps"])))

    def dominant(prof):
        """The sweep kernel with the largest share of the step: its HBM bytes
        per launch / its mean event-timed launch duration."""
        best = max(prof.items(), key=lambda kv: sum(ms for _, ms in kv[1]))
        di, lst = best
        nb = sum(b for b, _ in lst) / len(lst)
        ms = sum(t for _, t in lst) / len(lst)
        share = sum(t for _, t in lst) / max(sum(t for l2 in prof.values() for _, t in l2), 1e-30)
        return di, nb, ms, share

    dom_di, dom_bytes, dom_ms, dom_share = dominant(acc["prof"])
    dom_ms = max_over_ranks(dom_ms)
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    all_achieved = max_over_ranks(float(acc["sweep_bytes"])) / compute_s / 1e9

    # e2e: each process's initial rank blocks (|0...0> at layout phase 0) from
    # pinned host memory through run_plan(initial=...), final blocks back to
    # pinned host memory
    torch.cuda.synchronize()
    d = plan.d
    L = d - plan.g
    e2e = None
    nbytes = 16 * (rows << L)
    # pinned host buffers of all processes of the node must fit in half its RAM:
    # separate in/out buffers, else one buffer whose output feeds the next step
    # (any normalised state is a valid input), else no e2e line
    host_ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    nbuf = 2 if 2 * local_world * nbytes <= host_ram // 2 else (1 if local_world * nbytes <= host_ram // 2 else 0)
    if nbuf and nbytes <= E2E_HOST_BYTES and args.e2e_steps > 0:
        host_in = torch.zeros((rows, 1 << L), dtype=torch.complex128).pin_memory()
        if rank == 0:
            host_in[0, 0] = 1.0
        host_out = torch.empty((rows, 1 << L), dtype=torch.complex128).pin_memory() if nbuf == 2 else host_in
        run_plan(plan, initial=host_in, out=host_out).wait()  # warm
        barrier()
        t0 = time.perf_counter()
        prev = None
        for _ in range(args.e2e_steps):
            # two circuits in flight: this one's upload overlaps the previous
            # one's compute and download (every copy still runs every step)
            r = run_plan(plan, initial=host_in, out=host_out, wait=nbuf == 1 or not E2E_PIPELINE)
            if prev is not None:
                prev.wait()
            prev = r
            if nbuf == 1:
                r.wait()  # one host buffer: the next upload reads what this download writes
        prev.wait()
        del prev, r
        torch.cuda.synchronize()
        barrier()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / args.e2e_steps)
        e2e = {"value": total_bytes / e2e_s / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": world * 16 * (rows << L), "d2h_bytes_per_step": world * 16 * (rows << L),
               "bytes_note": "whole job: every process copies its own rank blocks in and out"
                             + ("" if nbuf == 2 else "; one pinned buffer per process, each step's output is the next input"),
               "ms_per_step": 1e3 * e2e_s}

    # sub-measurements at N=1 (timed the same way, reported beside the headline):
    # the same circuit with every sweep a full dense pass, and QV-30 (cfg3's
    # family on one GPU), whose sweeps are FP64-heavy
    subs = {}
    if world == 1 and args.workload == "qft" and args.sub_steps > 0:
        executor.SPARSE_START = False
        warm(plan, 3)
        a2 = timed(plan, args.sub_steps)
        executor.SPARSE_START = True
        subs["dense_passes"] = {
            "note": "same plan, sparse start off: every sweep reads and writes the whole state",
            "circuit_ms": 1e3 * a2["elapsed"] / args.sub_steps,
            "value": total_bytes * args.sub_steps / a2["elapsed"] / 1e9,
            "sweeps_frac": a2["sweep_bytes"] / a2["compute_s"] / 1e9 / peak}
        qvp = load_plan("qv30_h30-12")
        # first run with nothing cached (program compile + NVRTC of every
        # sweep kernel, pipelined with the sweeps it already has): the latency
        # a caller that sees the circuit once pays
        import tempfile

        from paper_2509_14098_b200 import jit as jitmod

        cold_dir = tempfile.mkdtemp(prefix="svb_jit_cold_")
        saved = jitmod.CACHE_DIR
        jitmod.CACHE_DIR = Path(cold_dir)
        jitmod._mem_cache.clear()
        executor._compile_cache.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        del_ = run_plan(qvp)
        torch.cuda.synchronize()
        first_run_s = time.perf_counter() - t0
        jitmod.CACHE_DIR = saved
        del del_
        warm(qvp, 2)
        a3 = timed(qvp, max(1, args.sub_steps // 3))
        k3 = max(1, args.sub_steps // 3)
        di3, b3, ms3, sh3 = dominant(a3["prof"])
        subs["qv30_h30-12"] = {
            "circuit_ms": 1e3 * a3["elapsed"] / k3, "value": plan_bytes(qvp) * k3 / a3["elapsed"] / 1e9,
            "sweeps_per_step": a3["sweeps"] // k3,
            "sweeps_hbm_frac": a3["sweep_bytes"] / a3["compute_s"] / 1e9 / peak,
            "dominant": {"sweep": di3, "launch_ms": ms3, "hbm_frac": b3 / (ms3 / 1e3) / 1e9 / peak,
                         "share_of_sweep_time": sh3, "fp64": fp64_roofline(qvp, di3, ms3)},
            "compile_ms": 1e3 * a3["stats"].compile_seconds,
            "first_run_ms": 1e3 * first_run_s,
            "first_run_note": "wall time of the first run_plan with empty JIT caches (plan compile + NVRTC of "
                              f"every kernel on {os.cpu_count()} host cores, overlapped with the sweeps)",
            "fp64_all_sweeps": fp64_all_sweeps(qvp, a3["prof"], a3["compute_s"] / k3, k3)}

    traffic = fp64 = None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            entry = json.loads(prof.read_text()).get(name) or {}
            if entry.get("rev") == TRAFFIC_REV and entry.get("sweep") == dom_di:  # same code, same kernel
                traffic = entry.get("bytes_per_launch")
                fp64 = entry.get("fp64_pipe_pct")
        except Exception:
            traffic = fp64 = None

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": name, "qubits": plan.d, "ranks": 1 << plan.g,
                   "hierarchy": [plan.d - plan.g, 12], "apply_fused": fused,
                   "exchanges": [len(t.payload["swaps"]) for t in plan.tasks if t.kind == "Exchange"],
                   "parallelism": f"state-vector sharding over {n} GPU(s)",
                   "l2": f"state {16 << plan.d >> 30} GiB >> 126 MB L2 (no flush needed)",
                   "value_def": "SURVEY 8(d) algorithmic bytes, 32 B x 2^d per ApplyFused leaf, / circuit time: "
                                "an effective rate comparable with the reference arm; the bytes the sweeps "
                                "actually move are in roofline.all_sweeps",
                   "circuits_in_flight": in_flight(plan)},
        "circuit_ms": 1e3 * elapsed / args.steps,
        "gates_per_s": sum(len(t.payload["gates"]) for t in plan.tasks if t.kind == "ApplyFused")
                        * args.steps / elapsed,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": f"sweep {dom_di} (NVRTC-specialised svb_jit_*), the largest share of the step",
                     "peak_source": f"{peak_kind} hbm_gbs (copy bandwidth, burst)",
                     "bytes_per_launch": dom_bytes, "launch_ms": dom_ms, "share_of_sweep_time": dom_share,
                     "bytes_note": "HBM bytes the launch must move: 16 B per amplitude read + 16 B per "
                                   "amplitude written (sparse |0...0>-start sweeps read only the support)",
                     "per_sweep_ms": {str(di): round(sum(t for _, t in lst) / len(lst), 4)
                                      for di, lst in sorted(acc["prof"].items())},
                     "all_sweeps": {"achieved": all_achieved, "frac": all_achieved / peak,
                                    "bytes_per_step": acc["sweep_bytes"] // args.steps,
                                    "launches_per_step": sweeps // args.steps,
                                    "sweep_ms_per_step": 1e3 * compute_s / args.steps},
                     "fp64_pipe_pct": fp64,
                     "frac_dram": (traffic / (dom_ms / 1e3) / 1e9 / peak) if traffic else None,
                     "frac_dram_note": "ncu DRAM bytes (read + write) of this kernel per launch / its event-timed "
                                       "launch / peak; traffic from profiles/traffic.json (same code revision)"},
        "e2e": e2e,
        "gpu_launches": launches,
        "compile_ms": 1e3 * stats.compile_seconds,
        "exchange_ms": 1e3 * stats.exchange_seconds,
        "clocks": clk.summary(),
    }
    if subs:
        line["sub"] = subs
    if world > 1:
        swap_s = max_over_ranks(stats.swap_seconds)
        line["nvlink"] = {
            "bytes_per_direction_per_step": stats.nvlink_bytes,
            "swap_ms": 1e3 * swap_s,
            "gbs_per_direction": stats.nvlink_bytes / swap_s / 1e9 if swap_s else None,
            "peak_gbs_per_direction": 900.0,
            "note": "per GPU: bytes it sends (= receives) over NVLink per circuit / event-timed swap kernels "
                    "(max over ranks); overlapped chunks share HBM with the sweeps",
        }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_line()
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": repr(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
