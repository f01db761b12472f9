"""Gate fusion (program.fuse_prims): SU(4)-style pair blocks fuse into one
4x4; pair blocks of bit flips and phases whose flips cancel (QAOA's cx rz cx)
become phases; the block's matrix is preserved either way."""

import numpy as np

from paper_2509_14098_b200 import program as prog


def _cx(c, t):
    return prog.Dense1(t, prog._X.copy(), {c: 1}, perm=True)


def _mat(prims, a, b):
    m = np.eye(4, dtype=np.complex128)
    for p in prims:
        m = prog._embed2(p, a, b) @ m
    return m


def test_cx_rz_cx_becomes_phases():
    a, b = 7, 3  # control a, target b
    th = 0.37
    prims = [_cx(a, b), prog.Factor((b,), np.exp(1j * th)), prog.Factor((), np.exp(-0.5j * th)), _cx(a, b)]
    out = prog.fuse_prims(prims)
    assert all(isinstance(p, prog.Factor) for p in out), out
    assert np.allclose(_mat(out, a, b), _mat(prims, a, b), atol=1e-15)


def test_flips_that_do_not_cancel_stay_flips():
    a, b = 7, 3
    prims = [_cx(a, b), prog.Factor((b,), 1j)]
    out = prog.fuse_prims(prims)
    assert any(isinstance(p, prog.Dense1) and p.perm for p in out)
    assert np.allclose(_mat(out, a, b), _mat(prims, a, b), atol=1e-15)


def test_global_controls_keep_the_flips():
    """A flip with a rank-global control resolves differently per device:
    the block is left alone so every device plans the same schedule."""
    a, b = 7, 3
    g = prog.Dense1(b, prog._X.copy(), {a: 1}, perm=True, gctl=True)
    prims = [g, prog.Factor((b,), 1j), prog.Dense1(b, prog._X.copy(), {a: 1}, perm=True, gctl=True)]
    out = prog.fuse_prims(prims)
    assert sum(isinstance(p, prog.Dense1) for p in out) == 2


def test_two_dense_gates_on_a_pair_fuse():
    a, b = 5, 1
    rng = np.random.default_rng(3)
    u = [np.linalg.qr(rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2)))[0] for _ in range(2)]
    prims = [prog.Dense1(a, u[0], {}), _cx(a, b), prog.Dense1(b, u[1], {})]
    out = prog.fuse_prims(prims)
    assert len(out) == 1 and isinstance(out[0], prog.Dense2)
    assert np.allclose(out[0].m, _mat(prims, out[0].a, out[0].b), atol=1e-14)
