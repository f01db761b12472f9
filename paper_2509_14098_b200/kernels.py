"""Inner kernel plugin: GPU twin of ``svpart.kernels`` (``kernels/__init__.py:39-60``).

``apply_gate(blocks, matrix, bits)`` / ``apply_diagonal(blocks, diag, bits)``
mutate (ranks, 2^L) complex128 blocks in place; ``bits`` are local positions
in gate-slot order, 0 = most significant.  ``blocks`` may be a CUDA tensor
(used in place) or a C-contiguous numpy array (copied to the GPU, updated,
copied back in place -- the reference's calling convention).  ``BACKEND`` is
always ``"b200"``: there is no CPU implementation behind this module.

The compiled core of the reference caps gates at 6 qubits and raises
ValueError on a shape mismatch (``_core.pyx:14-15``); the dispatcher routes
wider gates elsewhere (``kernels/__init__.py:41-42``).  Here gates up to 10
qubits run on the device; ``core_apply_gate`` keeps the strict 6-qubit
contract of ``_core.apply_gate``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native

BACKEND = "b200"
MAX_WIDTH = 10
CORE_MAX_WIDTH = 6


def _device_blocks(blocks):
    if isinstance(blocks, torch.Tensor):
        if not blocks.is_cuda or blocks.dtype != torch.complex128 or not blocks.is_contiguous():
            raise ValueError("blocks must be a contiguous complex128 CUDA tensor")
        return blocks, None
    if not isinstance(blocks, np.ndarray) or blocks.dtype != np.complex128 or not blocks.flags.c_contiguous:
        raise ValueError("blocks must be a C-contiguous complex128 array")
    return torch.from_numpy(blocks).cuda(), blocks


def _call(fn_name: str, blocks, table, bits, width: int):
    lib = _native.load()
    dev, host = _device_blocks(blocks)
    if dev.dim() != 2:
        raise ValueError("blocks must be 2-D (ranks, 2^L)")
    t = torch.from_numpy(np.array(table, dtype=np.complex128, copy=True).reshape(-1)).to(dev.device)
    arr, ptr = _native.i64_array(list(bits))
    dim = int(np.asarray(table).shape[0])
    rc = getattr(lib, fn_name)(dev.data_ptr(), dev.shape[0], dev.shape[1], t.data_ptr(), dim,
                               ptr, len(arr), width, torch.cuda.current_stream(dev.device).cuda_stream)
    _native.check(rc, fn_name)
    if host is not None:
        host[...] = dev.cpu().numpy()


def apply_gate(blocks, matrix, bits) -> None:
    """Apply a dense p-qubit gate in place; bit 0 is the local MSB."""
    _call("svb_apply_gate", blocks, matrix, bits, MAX_WIDTH)


def apply_diagonal(blocks, diag, bits) -> None:
    """Apply a diagonal p-qubit gate in place; bit 0 is the local MSB."""
    _call("svb_apply_diagonal", blocks, diag, bits, MAX_WIDTH)


def core_apply_gate(blocks, matrix, bits) -> None:
    """Strict twin of ``_core.apply_gate`` (ValueError above 6 qubits)."""
    _call("svb_apply_gate", blocks, matrix, bits, CORE_MAX_WIDTH)


def core_apply_diagonal(blocks, diag, bits) -> None:
    _call("svb_apply_diagonal", blocks, diag, bits, CORE_MAX_WIDTH)
