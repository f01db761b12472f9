"""INTEGRATION.md section 1 executed: the proposed executor switch is
appended to a copy of the reference's svpart/executor.py, and with
SVPART_EXECUTOR=b200 the reference package and its CLI resolve run_plan,
gather, compare and the exception classes to this executor.  CPU only
(the reference source exists in the build container, not on the GPU box)."""

import os
import re
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import ROOT

REF = Path("/root/reference/pkg/src/svpart")


@pytest.mark.skipif(not REF.exists(), reason="reference source not present")
def test_reference_executor_switch(tmp_path):
    text = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"```python\n(# svpart/executor.py \(proposed addition.*?)```", text, re.S).group(1)
    pkg = tmp_path / "svpart"
    shutil.copytree(REF, pkg, ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    (pkg / "executor.py").write_text((pkg / "executor.py").read_text() + "\n" + block)
    probe = f"""
import sys
sys.path[:0] = [{str(tmp_path)!r}, {str(ROOT)!r}]
import svpart, svpart.executor as ex, svpart.cli as cli
import paper_2509_14098_b200 as b200
assert svpart.run_plan is b200.run_plan and ex.run_plan is b200.run_plan
assert ex.gather is b200.gather and ex.compare is b200.compare
for name in ("TooLarge", "PlanInvalid", "NonUnitaryDrift", "DimensionMismatch"):
    assert getattr(ex, name) is getattr(b200, name), name
# the CLI maps the executor's errors through the rebound names (cli.py:297-310)
def boom(*a, **k):
    raise b200.TooLarge("state too large for this test")
ex.run_plan = boom
open({str(tmp_path / 'c.qasm')!r}, "w").write("OPENQASM 2.0;\\nqreg q[3];\\nh q[0];\\ncx q[0],q[1];\\n")
rc = cli.main(["run", {str(tmp_path / 'c.qasm')!r}, "--ranks", "2"])
assert rc == cli.EXIT_PARTITION, rc
print("rebind ok")
"""
    env = dict(os.environ, SVPART_EXECUTOR="b200", PYTHONPATH="")
    r = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0 and "rebind ok" in r.stdout, r.stderr[-2000:]
