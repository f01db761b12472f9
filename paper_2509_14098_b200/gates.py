"""Gate table for the state-vector executor.

The executor must reproduce the reference's numerics bit-for-bit at the
matrix level, so every entry here is built from the same closed forms the
reference documents (``svpart/gates.py:20-121``):

* qubit 0 is the most significant Kronecker factor; slot i of a p-qubit gate
  addresses bit (p-1-i) of the 2^p matrix index; controls come first;
* ``p(a) = diag(1, e^{-ia})`` and ``cp(a) = diag(1, 1, 1, e^{-ia})`` (the
  reference's sign convention, ``gates.py:98-101``);
* a gate is "diagonal" iff every off-diagonal magnitude is below 1e-15
  (``gates.py:17``, ``:124-126``), so e.g. ``rx(0)`` counts as diagonal.

Matrices are cached per (kind, params) and returned read-only.
"""

from __future__ import annotations

import cmath
import math
from dataclasses import dataclass, field

import numpy as np

DIAG_TOL = 1e-15

# kind -> (parameter count, qubit count, control slots); mirrors
# svpart/gates.py:20-40 (GATE_SIGNATURES)
SIGNATURES: dict[str, tuple[int, int, tuple[int, ...]]] = {
    "id": (0, 1, ()),
    "h": (0, 1, ()),
    "x": (0, 1, ()),
    "y": (0, 1, ()),
    "z": (0, 1, ()),
    "s": (0, 1, ()),
    "sdg": (0, 1, ()),
    "t": (0, 1, ()),
    "tdg": (0, 1, ()),
    "rx": (1, 1, ()),
    "ry": (1, 1, ()),
    "rz": (1, 1, ()),
    "p": (1, 1, ()),
    "u": (3, 1, ()),
    "cx": (0, 2, (0,)),
    "cz": (0, 2, (0,)),
    "cp": (1, 2, (0,)),
    "swap": (0, 2, ()),
    "ccx": (0, 3, (0, 1)),
}
GATE_SIGNATURES = SIGNATURES


@dataclass(frozen=True)
class Gate:
    """A concrete gate: matrix plus the structural flags the executor reads."""

    kind: str
    params: tuple[float, ...]
    matrix: np.ndarray = field(repr=False, compare=False)
    controls: frozenset[int]
    is_diagonal: bool

    @property
    def num_qubits(self) -> int:
        return self.matrix.shape[0].bit_length() - 1

    # reference spelling (GateTensor.control_dims)
    @property
    def control_dims(self) -> frozenset[int]:
        return self.controls


def _rot_pair(theta: float) -> tuple[float, float]:
    return math.cos(theta / 2), math.sin(theta / 2)


def _one_qubit(kind: str, params: tuple[float, ...]) -> list[list[complex]]:
    r = math.sqrt(2)
    if kind == "id":
        return [[1, 0], [0, 1]]
    if kind == "h":
        return [[1 / r, 1 / r], [1 / r, -1 / r]]
    if kind == "x":
        return [[0, 1], [1, 0]]
    if kind == "y":
        return [[0, -1j], [1j, 0]]
    if kind == "z":
        return [[1, 0], [0, -1]]
    if kind == "s":
        return [[1, 0], [0, 1j]]
    if kind == "sdg":
        return [[1, 0], [0, -1j]]
    if kind == "t":
        return [[1, 0], [0, cmath.exp(1j * math.pi / 4)]]
    if kind == "tdg":
        return [[1, 0], [0, cmath.exp(-1j * math.pi / 4)]]
    if kind == "rx":
        c, s = _rot_pair(params[0])
        return [[c, -1j * s], [-1j * s, c]]
    if kind == "ry":
        c, s = _rot_pair(params[0])
        return [[c, -s], [s, c]]
    if kind == "rz":
        th = params[0]
        return [[cmath.exp(-1j * th / 2), 0], [0, cmath.exp(1j * th / 2)]]
    if kind == "p":
        return [[1, 0], [0, cmath.exp(-1j * params[0])]]
    if kind == "u":
        th, ph, lam = params
        c, s = _rot_pair(th)
        return [
            [c, -cmath.exp(1j * lam) * s],
            [cmath.exp(1j * ph) * s, cmath.exp(1j * (ph + lam)) * c],
        ]
    raise KeyError(kind)


def _matrix(kind: str, params: tuple[float, ...]) -> np.ndarray:
    if kind in ("cx", "cz", "cp", "ccx", "swap"):
        if kind == "swap":
            m = np.eye(4, dtype=np.complex128)
            m[[1, 2]] = m[[2, 1]]
            return m
        n = 8 if kind == "ccx" else 4
        m = np.eye(n, dtype=np.complex128)
        if kind in ("cx", "ccx"):
            m[n - 2:, n - 2:] = np.array([[0, 1], [1, 0]], dtype=np.complex128)
        elif kind == "cz":
            m[3, 3] = -1
        else:
            m[3, 3] = cmath.exp(-1j * params[0])
        return m
    return np.array(_one_qubit(kind, params), dtype=np.complex128)


def _diagonal(m: np.ndarray) -> bool:
    off = m[~np.eye(m.shape[0], dtype=bool)]
    return bool(np.all(np.abs(off) < DIAG_TOL))


_cache: dict[tuple[str, tuple[float, ...]], Gate] = {}


def gate(kind: str, params=()) -> Gate:
    """Concrete gate for (kind, params); KeyError/ValueError like the reference."""
    params = tuple(float(p) for p in params)
    key = (kind, params)
    hit = _cache.get(key)
    if hit is not None:
        return hit
    if kind not in SIGNATURES:
        raise KeyError(kind)
    npar, _, ctl = SIGNATURES[kind]
    if len(params) != npar:
        raise ValueError(f"{kind} takes {npar} parameter(s), got {len(params)}")
    m = np.ascontiguousarray(_matrix(kind, params), dtype=np.complex128)
    m.setflags(write=False)
    g = Gate(kind=kind, params=params, matrix=m, controls=frozenset(ctl), is_diagonal=_diagonal(m))
    _cache[key] = g
    return g


# reference spelling
gate_tensor = gate
