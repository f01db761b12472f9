"""The reference arm of bench.py (--impl reference): one copy of the
single-threaded reference circuit per host core, one JSON line with the
contract's keys (run here on a small sample plan and two cores)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_line():
    if not any((ROOT / "oracle" / "_ref").glob("_core*.so")) and not (ROOT / "oracle" / "libsvoracle.so").exists():
        pytest.skip("oracle not built")
    env = dict(os.environ, SVB200_REF_CORES="2", SVB200_REF_SAMPLE="qft20_h18-12")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["cpu_baseline"]["cores"] == 2 and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["steps"] == 1 and line["warmup"] == 3
