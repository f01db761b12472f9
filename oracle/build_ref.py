"""Compile the reference's own Cython kernel (svpart/kernels/_core.pyx) into
oracle/_ref/ -- TEST INFRASTRUCTURE ONLY.

The source is read where it lies under /root/reference (never copied into
the repository); the generated C and the object files go to a temporary
directory and only the extension module lands in oracle/_ref/ (git-ignored,
shipped to the GPU box with the snapshot).  The module is importable as
``_core`` with oracle/_ref on sys.path and exposes the reference's exact
``apply_gate`` / ``apply_diagonal`` (``_core.pyx:7-9``, ``:63-65``).

Recipe = what the reference's setup.py does (setup.py:10-25): cythonize with
language_level=3 and numpy headers, compile with the interpreter's flags.
"""

from __future__ import annotations

import argparse
import shutil
import subprocess
import sys
import sysconfig
import tempfile
from pathlib import Path


def build(src: Path, out: Path) -> Path:
    import numpy
    from Cython.Build import cythonize  # noqa: F401  (presence check)

    out.mkdir(parents=True, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        pyx = tmp / "_core.pyx"
        shutil.copyfile(src, pyx)  # stays in the temp dir
        c_file = tmp / "_core.c"
        subprocess.run(
            [sys.executable, "-m", "cython", "-3", str(pyx), "-o", str(c_file)],
            check=True,
        )
        ext = sysconfig.get_config_var("EXT_SUFFIX")
        target = out / f"_core{ext}"
        inc = sysconfig.get_paths()["include"]
        subprocess.run(
            [
                "gcc", "-O2", "-fPIC", "-shared", "-fwrapv",
                "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION",
                f"-I{inc}", f"-I{numpy.get_include()}",
                str(c_file), "-o", str(target),
            ],
            check=True,
        )
    return target


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default="/root/reference/pkg/src/svpart/kernels/_core.pyx")
    ap.add_argument("--out", default=str(Path(__file__).resolve().parent / "_ref"))
    a = ap.parse_args()
    print(build(Path(a.src), Path(a.out)))
