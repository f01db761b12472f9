"""Build libsvb200.so (the C-ABI CUDA library) in-tree for sm_100a.

    python -m paper_2509_14098_b200._build          # build if stale
    python -m paper_2509_14098_b200._build --force

The library is written next to this file so it travels with the repo
snapshot to the GPU box (a JIT cache under ~/.cache would not).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libsvb200.so"
SOURCES = ["gate_kernels.cu", "sweep.cu", "layout.cu", "reduce.cu", "jit.cu", "peer.cu", "cdf.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("common.cuh")) + [INCLUDE / "svb200.h"]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    objdir = ROOT / "build" / "svb200"
    objdir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    common = [
        nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
        "-I", str(INCLUDE), "-I", str(CSRC), "--expt-relaxed-constexpr",
    ]
    if verbose:
        common += ["-Xptxas", "-v"]
    objs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        cmd = common + ["-c", str(CSRC / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    build_native_host(force=True)
    return LIB


NATIVE_HOST_SRC = ROOT / "native_host" / "svb_run.cpp"
NATIVE_HOST = ROOT / "native_host" / "svb_run"


def build_native_host(force: bool = False) -> Path:
    """native_host/svb_run: the C++ host that runs a program file
    (program_file.py) through include/svb200.h, without Python."""
    if not force and NATIVE_HOST.exists() and NATIVE_HOST.stat().st_mtime > max(
            NATIVE_HOST_SRC.stat().st_mtime, LIB.stat().st_mtime):
        return NATIVE_HOST
    cmd = [_nvcc(), "-std=c++17", "-O2", "-I", str(INCLUDE), str(NATIVE_HOST_SRC), "-o", str(NATIVE_HOST),
           "-L", str(PKG), "-lsvb200", "-lcudart", "-Xlinker", f"-rpath,$ORIGIN/../{PKG.name}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"native host build failed:\n{r.stderr}")
    return NATIVE_HOST


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)
