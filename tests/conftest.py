import gzip
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def grid_docs():
    with gzip.open(GOLDEN / "grid.json.gz", "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def grid_states():
    return dict(np.load(GOLDEN / "grid_states.npz"))


@pytest.fixture(scope="session")
def cfg1_docs():
    with gzip.open(GOLDEN / "cfg1.json.gz", "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def cfg1_fp():
    return dict(np.load(GOLDEN / "cfg1_fp.npz"))


def plan_from_doc(doc):
    from paper_2509_14098_b200.plan import from_json

    return from_json(json.dumps(doc))


@pytest.fixture(scope="session")
def family_docs():
    """Benchmark-family plans (QV / QAOA / supremacy / QFT from |x>) at D > K
    with the reference's fingerprints (tests/golden/make_golden.py --families)."""
    with gzip.open(GOLDEN / "families.json.gz", "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def family_fp():
    return dict(np.load(GOLDEN / "families_fp.npz"))


def family_initial(doc):
    """The dense initial state of a family case (None: |0...0>)."""
    x = doc.get("initial_basis")
    if x is None:
        return None
    v = np.zeros(1 << doc["plan"]["d"], dtype=np.complex128)
    v[x] = 1.0
    return v


def check_fingerprint(flat, fp, name, seed, tol=1e-10):
    """Compare flat rank-block storage with the reference's fingerprint:
    sampled amplitudes, the plain and a random-phase weighted sum, the norm
    (make_golden.fingerprint: a storage permutation changes them)."""
    rng = np.random.default_rng(seed)
    n = flat.size
    idx = rng.choice(n, size=min(8192, n), replace=False)
    idx = np.sort(idx)
    assert np.array_equal(idx, fp[name + "::idx"]), name
    w = np.exp(2j * np.pi * rng.random(n))
    err = float(np.max(np.abs(flat[idx] - fp[name + "::amps"])))
    assert err < tol, (name, "amps", err)
    assert abs(flat.sum() - fp[name + "::sum"][0]) < 1e-8, (name, "sum")
    assert abs((w * flat).sum() - fp[name + "::wsum"][0]) < 1e-8, (name, "wsum")
    assert abs(np.vdot(flat, flat).real - fp[name + "::norm"][0]) < 1e-10, (name, "norm")
    return err
