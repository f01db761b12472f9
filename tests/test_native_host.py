"""The native C++ host (native_host/svb_run.cpp): a
compiled device program written by program_file.export plus the plan JSON,
run without Python through include/svb200.h."""

import json
import subprocess

import numpy as np
import pytest

from conftest import ROOT, plan_from_doc

HOST = ROOT / "native_host" / "svb_run"


def test_program_file_round_trip(tmp_path):
    import struct

    from paper_2509_14098_b200 import plan as planmod, program as prog, program_file

    plan = planmod.load(str(ROOT / "plans" / "qft20_h18-12.json.gz"))
    path = program_file.export(plan, tmp_path / "cfg1")
    secs = program_file.read(path)
    d, g, L, D, rows, n_fused, sparse, nsteps, ndescs, nkernels, unit = struct.unpack("<11i", secs["HEAD"])
    assert (d, g, L, D, rows) == (20, 2, 18, 20, 4)
    assert n_fused == sum(1 for t in plan.tasks if t.kind == "ApplyFused")
    assert len(secs["DESC"]) == ndescs * prog.DESC_DTYPE.itemsize and nkernels == ndescs
    assert sparse == 1
    assert json.loads((tmp_path / "cfg1.plan.json").read_text())["d"] == 20


def test_native_host_usage():
    assert HOST.exists(), "build() compiles native_host/svb_run"
    r = subprocess.run([str(HOST)], capture_output=True, text=True)
    assert r.returncode == 1 and "usage" in r.stderr


def _run(plan, tmp_path, name):
    from paper_2509_14098_b200 import program_file

    path = program_file.export(plan, tmp_path / name)
    out = tmp_path / f"{name}.bin"
    r = subprocess.run([str(HOST), str(path), str(tmp_path / f"{name}.plan.json"), str(out)],
                       capture_output=True, text=True, timeout=600)
    return r, out


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["cfg1", "qv20_h18-12", "qaoa20_h18-12"])
def test_native_host_matches_python_bit_for_bit(tmp_path, which, family_docs):
    from paper_2509_14098_b200 import plan as planmod, run_plan

    if which == "cfg1":
        plan = planmod.load(str(ROOT / "plans" / "qft20_h18-12.json.gz"))
    else:
        plan = plan_from_doc(family_docs[which]["plan"])
    r, out = _run(plan, tmp_path, which)
    assert r.returncode == 0, r.stderr
    got = np.fromfile(out, dtype=np.complex128).reshape(1 << plan.g, -1)
    want = run_plan(plan).state.blocks.cpu().numpy()
    assert np.array_equal(got, want), float(np.max(np.abs(got - want)))


@pytest.mark.gpu
def test_native_host_rejects_protocol_errors(tmp_path, grid_docs):
    """Reordered tasks (reference test_executor.py:146-152): PlanInvalid, exit code 2."""
    from paper_2509_14098_b200 import program_file
    from paper_2509_14098_b200.plan import ExecutionPlan

    plan = plan_from_doc(next(d for d in grid_docs if d["name"] == "ghz3-2")["plan"])
    path = program_file.export(plan, tmp_path / "ghz")
    doc = json.loads((tmp_path / "ghz.plan.json").read_text())
    doc["tasks"][1], doc["tasks"][5] = doc["tasks"][5], doc["tasks"][1]
    (tmp_path / "ghz.plan.json").write_text(json.dumps(doc))
    r = subprocess.run([str(HOST), str(path), str(tmp_path / "ghz.plan.json"), str(tmp_path / "o.bin")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "PlanInvalid" in r.stderr, r.stderr
