"""The C-ABI library loads and exports every symbol include/svb200.h declares (no GPU needed)."""

import ctypes
import re
from pathlib import Path

from paper_2509_14098_b200 import _native

HEADER = Path(__file__).resolve().parent.parent / "include" / "svb200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(svb_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(_native.EXPORTS) <= set(names)


def test_abi_struct_sizes_match():
    lib = _native.load()  # raises on mismatch
    assert lib.svb_abi_version() == 1


def test_validation_errors_without_gpu():
    lib = _native.load()
    import numpy as np

    bits, ptr = _native.i64_array([0])
    # width/shape mismatch is rejected before any device work (_core.pyx:14-15)
    rc = lib.svb_apply_gate(None, 1, 4, None, 4, ptr, 1, 6, None)
    assert rc == _native.SVB_EINVAL
    assert b"shape" in lib.svb_last_error()
    rc = lib.svb_apply_gate(None, 1, 6, None, 2, ptr, 1, 6, None)  # n not a power of two
    assert rc == _native.SVB_EINVAL
