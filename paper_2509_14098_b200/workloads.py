"""Synthetic circuits of the benchmark shapes, emitted as OpenQASM 2.0 text.

The reference ships ghz/dj/qft/qpe/ising/su2random/vqc emitters
(``svpart/circuits.py:19-100``); the BASELINE configurations also name a
quantum-volume, a QAOA MaxCut and a Google-style random circuit, which the
reference does not have.  These emitters use only the reference's gate set
(``gates.py:20-40``) and write angles with ``repr(float(x))`` because the
reference tokenizer rejects numpy-2 scalar reprs (``qasm.py:84-104``).
Every family is deterministic given (d, seed).

``qft`` reproduces the reference family exactly (same text) so plans for
QFT-n match ``svpart.circuits.qft(n)`` gate for gate.
"""

from __future__ import annotations

import math

import numpy as np


def _head(d: int) -> list:
    return ["OPENQASM 2.0;", 'include "qelib1.inc";', f"qreg q[{d}];"]


def _f(x) -> str:
    return repr(float(x))


def qft(d: int, seed: int = 0) -> str:
    """Textbook QFT without final-swap elision: h, cp(pi/2^k) ladders, swaps."""
    out = _head(d)
    for i in range(d):
        out.append(f"h q[{i}];")
        for j in range(i + 1, d):
            out.append(f"cp(pi/{1 << (j - i)}) q[{j}],q[{i}];")
    for i in range(d // 2):
        out.append(f"swap q[{i}],q[{d - 1 - i}];")
    return "\n".join(out) + "\n"


def quantum_volume(d: int, seed: int = 0, depth: int | None = None) -> str:
    """Quantum-volume model circuit: `depth` layers of random SU(4) on a random pairing.

    Each SU(4) is emitted in the KAK-like form u,u,cx,u,u,cx,u,u,cx,u,u with
    angles uniform in [0, 2pi) (11 gates per block).
    """
    depth = d if depth is None else depth
    rng = np.random.default_rng(seed)
    out = _head(d)
    for _ in range(depth):
        perm = rng.permutation(d)
        for k in range(d // 2):
            a, b = int(perm[2 * k]), int(perm[2 * k + 1])
            for rep in range(4):
                for q in (a, b):
                    th, ph, la = rng.uniform(0, 2 * math.pi, size=3)
                    out.append(f"u({_f(th)},{_f(ph)},{_f(la)}) q[{q}];")
                if rep < 3:
                    out.append(f"cx q[{a}],q[{b}];")
    return "\n".join(out) + "\n"


def near_regular_graph(n: int, degree: int = 3, seed: int = 0) -> list:
    """Random simple graph with every vertex of the given degree, except one
    vertex of degree-1 when n*degree is odd (a 3-regular graph on an odd
    number of vertices does not exist)."""
    rng = np.random.default_rng(seed)
    want = [degree] * n
    if (n * degree) % 2:
        want[n - 1] = degree - 1
    for _attempt in range(1000):
        stubs = [v for v in range(n) for _ in range(want[v])]
        rng.shuffle(stubs)
        edges = set()
        ok = True
        for i in range(0, len(stubs), 2):
            a, b = stubs[i], stubs[i + 1]
            e = (min(a, b), max(a, b))
            if a == b or e in edges:
                ok = False
                break
            edges.add(e)
        if ok:
            return sorted(edges)
    raise RuntimeError("could not sample a simple near-regular graph")


def qaoa_maxcut(d: int, seed: int = 0, p: int = 4, degree: int = 3) -> str:
    """QAOA-p MaxCut: h layer, then p x (cx-rz(2 gamma)-cx per edge, rx(2 beta) layer)."""
    rng = np.random.default_rng(seed + 1)
    edges = near_regular_graph(d, degree, seed)
    out = _head(d)
    out += [f"h q[{i}];" for i in range(d)]
    for _ in range(p):
        gamma, beta = rng.uniform(0, math.pi, size=2)
        for a, b in edges:
            out.append(f"cx q[{a}],q[{b}];")
            out.append(f"rz({_f(2 * gamma)}) q[{b}];")
            out.append(f"cx q[{a}],q[{b}];")
        out += [f"rx({_f(2 * beta)}) q[{i}];" for i in range(d)]
    return "\n".join(out) + "\n"


def random_supremacy(d: int, seed: int = 0, depth: int = 20, rows: int | None = None) -> str:
    """Boixo-style random circuit on a rows x cols grid.

    Cycle 0 is a Hadamard layer; each of the `depth` cycles applies one of 8
    staggered CZ patterns (horizontal/vertical, even/odd columns or rows,
    two offsets) and, on qubits idle in this cycle that took part in a CZ in
    the previous cycle, a random single-qubit gate from {t, rx(pi/2),
    ry(pi/2)} different from that qubit's previous one (t first).
    """
    if rows is None:
        rows = int(math.isqrt(d))
        while d % rows:
            rows -= 1
    cols = d // rows
    rng = np.random.default_rng(seed)

    def q(r, c):
        return r * cols + c

    patterns = []
    for horiz in (True, False):
        for par in (0, 1):
            for off in (0, 1):
                pairs = []
                if horiz:
                    for r in range(rows):
                        if r % 2 != off:
                            continue
                        for c in range(par, cols - 1, 2):
                            pairs.append((q(r, c), q(r, c + 1)))
                else:
                    for c in range(cols):
                        if c % 2 != off:
                            continue
                        for r in range(par, rows - 1, 2):
                            pairs.append((q(r, c), q(r + 1, c)))
                patterns.append(pairs)
    order = [0, 4, 1, 5, 2, 6, 3, 7]
    out = _head(d)
    out += [f"h q[{i}];" for i in range(d)]
    last_gate = ["t_pending"] * d  # first single-qubit gate on a qubit is t
    prev_cz = set(range(d))
    for cyc in range(depth):
        pairs = patterns[order[cyc % 8]]
        busy = {x for pr in pairs for x in pr}
        for i in range(d):
            if i in busy or i not in prev_cz:
                continue
            if last_gate[i] == "t_pending":
                g = "t"
            else:
                choices = [x for x in ("t", "rx", "ry") if x != last_gate[i]]
                g = choices[int(rng.integers(0, len(choices)))]
            last_gate[i] = g
            if g == "t":
                out.append(f"t q[{i}];")
            else:
                out.append(f"{g}(pi/2) q[{i}];")
        for a, b in pairs:
            out.append(f"cz q[{a}],q[{b}];")
        prev_cz = busy
    return "\n".join(out) + "\n"


FAMILIES = {
    "qft": qft,
    "qv": quantum_volume,
    "qaoa": qaoa_maxcut,
    "supremacy": random_supremacy,
}


_SELF_INVERSE = {"id", "h", "x", "y", "z", "cx", "cz", "swap", "ccx"}
_SWAP_INV = {"t": "tdg", "tdg": "t", "s": "sdg", "sdg": "s"}
_NEG = {"rx", "ry", "rz", "p", "cp"}


def _inverse_line(line: str) -> str:
    """Inverse of one gate statement of the reference gate set."""
    stmt = line.strip().rstrip(";")
    head, _, args = stmt.partition(" ")
    name, _, par = head.partition("(")
    par = par.rstrip(")")
    if name in _SELF_INVERSE:
        return line
    if name in _SWAP_INV:
        return f"{_SWAP_INV[name]} {args};"
    if name in _NEG:
        return f"{name}(-({par})) {args};"
    if name == "u":  # u(t, f, l)^dagger = u(-t, -l, -f)
        t, f, lam = (x.strip() for x in par.split(","))
        return f"u(-({t}),-({lam}),-({f})) {args};"
    raise ValueError(f"no inverse for {name}")


def inverse(qasm: str) -> str:
    """U^dagger of a circuit: its gates inverted in reverse order."""
    lines = qasm.strip().splitlines()
    head = [ln for ln in lines if ln.startswith(("OPENQASM", "include", "qreg"))]
    body = [ln for ln in lines if ln not in head and ln.strip()]
    return "\n".join(head + [_inverse_line(ln) for ln in reversed(body)]) + "\n"


def mirror(qasm: str) -> str:
    """U followed by U^dagger: the exact output is |0...0> (a full-size known answer)."""
    lines = qasm.strip().splitlines()
    head = [ln for ln in lines if ln.startswith(("OPENQASM", "include", "qreg"))]
    body = [ln for ln in lines if ln not in head and ln.strip()]
    return "\n".join(head + body + [_inverse_line(ln) for ln in reversed(body)]) + "\n"


def basis_qft_amplitudes(d: int, x: int, y):
    """Closed form of the reference QFT (svpart/circuits.py:34-42) on |x>:
    amp(y) = 2^(-d/2) exp(-2 pi i x y / 2^d), qubit 0 the most significant bit."""
    xy = (np.asarray(y, dtype=np.int64) * x) & ((1 << d) - 1)
    return np.exp(-2j * np.pi * xy / (1 << d)) / (2 ** (d / 2))
