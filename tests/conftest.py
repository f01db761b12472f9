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
