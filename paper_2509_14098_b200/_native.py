"""ctypes binding of libsvb200.so (the C ABI declared in include/svb200.h).

There is no fallback: if the library is missing or fails to load, every
entry point raises NativeError.  Pointers are plain integers (torch
``data_ptr()``); streams are ``torch.cuda.Stream.cuda_stream`` integers.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import NativeError

LIB_PATH = Path(__file__).resolve().parent / "libsvb200.so"

SVB_OK, SVB_EINVAL, SVB_ECUDA, SVB_ERANGE = 0, 1, 2, 3

_c = ctypes
_vp, _i64, _i32, _int, _u32, _sz = _c.c_void_p, _c.c_int64, _c.c_int32, _c.c_int, _c.c_uint32, _c.c_size_t
_pi64 = _c.POINTER(_c.c_int64)
_pi32 = _c.POINTER(_c.c_int32)
_pd = _c.c_void_p

_SIGS = {
    "svb_abi_version": ([], _int),
    "svb_last_error": ([], _c.c_char_p),
    "svb_abi_sizes": ([_c.POINTER(_sz)] * 3, None),
    "svb_apply_gate": ([_vp, _i64, _i64, _vp, _i64, _pi64, _int, _int, _vp], _int),
    "svb_apply_diagonal": ([_vp, _i64, _i64, _vp, _i64, _pi64, _int, _int, _vp], _int),
    "svb_run_sweeps": ([_vp, _i64, _int, _vp, _vp, _int, _vp, _int, _vp], _int),
    "svb_bitswap": ([_vp, _int, _pi32, _pi32, _int, _vp], _int),
    "svb_pack_region": ([_vp, _i64, _int, _pi32, _int, _u32, _i64, _i64, _vp, _vp], _int),
    "svb_unpack_region": ([_vp, _i64, _int, _pi32, _int, _u32, _i64, _i64, _vp, _vp], _int),
    "svb_bitperm": ([_vp, _vp, _int, _pi32, _vp], _int),
    "svb_norm2": ([_vp, _i64, _vp, _vp], _int),
    "svb_compare_scratch_bytes": ([_i64], _sz),
    "svb_compare": ([_vp, _vp, _i64, _vp, _vp, _vp], _int),
    "svb_shard_scratch_bytes": ([_i64], _sz),
    "svb_shard_argmax": ([_vp, _vp, _i64, _c.c_uint64, _int, _pi32, _vp, _vp, _vp], _int),
    "svb_shard_maxdev": ([_vp, _vp, _i64, _c.c_double, _c.c_double, _vp, _vp, _vp], _int),
    "svb_jit_compile": ([_c.c_char_p, _c.c_char_p, _int, _c.POINTER(_c.c_char_p), _c.POINTER(_vp),
                         _c.POINTER(_sz), _c.c_char_p, _sz], _int),
    "svb_jit_free": ([_vp], None),
    "svb_jit_load": ([_c.c_char_p, _c.c_char_p, _c.POINTER(_vp)], _int),
    "svb_jit_launch_sweep": ([_vp, _vp, _vp, _vp, _vp, _int, _vp], _int),
    "svb_jit_launch_sweep_part": ([_vp, _vp, _vp, _vp, _vp, _int, _c.c_uint64, _c.c_uint64, _i64, _vp],
                                  _int),
    "svb_dev_alloc": ([_sz, _c.POINTER(_vp)], _int),
    "svb_dev_free": ([_vp], _int),
    "svb_ipc_handle": ([_vp, _vp], _int),
    "svb_ipc_open": ([_vp, _c.POINTER(_vp)], _int),
    "svb_ipc_close": ([_vp], _int),
    "svb_peer_swap_bulk": ([_vp, _vp, _int, _i64, _int, _pi32, _int, _vp, _vp, _vp, _vp, _int, _int, _int, _int,
                            _vp],
                           _int),
    "svb_stream_write_u32": ([_vp, _u32, _vp], _int),
    "svb_stream_wait_u32": ([_vp, _u32, _vp], _int),
    "svb_stream_create": ([_c.POINTER(_vp)], _int),
    "svb_gather_bits": ([_vp, _int, _pi32, _c.c_uint64, _i64, _vp, _vp], _int),
    "svb_region_move": ([_vp, _int, _pi32, _int, _u32, _u32, _vp], _int),
    "svb_cdf_chunk_elems": ([], _i64),
    "svb_probs_numpy": ([_vp, _int, _pi32, _vp, _vp], _int),
    "svb_deposit_scatter": ([_vp, _i64, _int, _pi32, _c.c_uint64, _vp, _vp], _int),
    "svb_pairwise_scratch_bytes": ([_int], _sz),
    "svb_pairwise_sum": ([_vp, _int, _vp, _vp, _vp], _int),
    "svb_div_scalar": ([_vp, _i64, _vp, _vp], _int),
    "svb_cdf_scratch_bytes": ([_i64], _sz),
    "svb_cdf_chunk_totals": ([_vp, _i64, _vp, _vp], _int),
    "svb_cdf_walk": ([_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "svb_cdf_search": ([_vp, _i64, _vp, _i64, _i64, _i64, _c.c_double, _vp, _i64, _i64, _vp, _vp], _int),
    "svb_copy": ([_vp, _vp, _i64, _int, _vp], _int),
    "svb_peer_swap": ([_vp, _vp, _int, _i64, _int, _pi32, _int, _vp, _vp, _vp, _vp, _int, _int, _vp], _int),
}

EXPORTS = tuple(_SIGS)

_lib = None
_load_error: str | None = None


def load():
    """Load the library once; raises NativeError with the reason on failure."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise NativeError(_load_error)
    path = os.environ.get("SVB200_LIB", str(LIB_PATH))
    try:
        lib = ctypes.CDLL(path)
    except OSError as e:
        _load_error = f"cannot load {path}: {e} (build with `python -m paper_2509_14098_b200._build`)"
        raise NativeError(_load_error) from e
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    _check_abi(lib)
    return lib


def _check_abi(lib) -> None:
    from .program import CTERM_DTYPE, DESC_DTYPE, OP_DTYPE

    a, b, c = _sz(), _sz(), _sz()
    lib.svb_abi_sizes(_c.byref(a), _c.byref(b), _c.byref(c))
    got = (a.value, b.value, c.value)
    want = (OP_DTYPE.itemsize, CTERM_DTYPE.itemsize, DESC_DTYPE.itemsize)
    if got != want:
        raise NativeError(f"ABI struct size mismatch: library {got}, python {want}")


def check(rc: int, what: str) -> None:
    if rc != SVB_OK:
        msg = load().svb_last_error().decode(errors="replace")
        if rc == SVB_EINVAL:
            raise ValueError(f"{what}: {msg}")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def i64_array(vals):
    arr = np.ascontiguousarray(np.asarray(vals, dtype=np.int64))
    return arr, arr.ctypes.data_as(_pi64)


def i32_array(vals):
    arr = np.ascontiguousarray(np.asarray(vals, dtype=np.int32))
    return arr, arr.ctypes.data_as(_pi32)
