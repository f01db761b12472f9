"""Memory and race self-check on the GPU (compute-sanitizer is closed on the
GPU pool): tools/selfcheck.py in a fresh process with bounds-checked
generated kernels, guard bands around the state and grid-shape variation."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bounds_guards_and_grid_determinism():
    env = dict(os.environ, SVB200_JIT_CHECK="1", SVB200_GUARD_AMPS="65536",
               SVB200_JIT_CACHE=str(ROOT / "build" / "jit_cache_check"))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "selfcheck.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0 and "0 mismatches" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])
