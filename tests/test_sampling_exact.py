"""The numpy-identical sampling algorithm (csrc/cdf.cu, sampling.py) restated
in numpy and checked against numpy itself on CPU: the complex absolute value,
the pairwise sum tree, and the exact sequential cumsum through integer ulp
increments per binade (with ties and binade crossings).  The GPU tests then
check the kernels against numpy (tests/test_sampling.py)."""

import math
from fractions import Fraction

import numpy as np
import pytest

from paper_2509_14098_b200.sampling import pairwise_combine


def fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def numpy_cabs(z):
    ax, ay = abs(z.real), abs(z.imag)
    big, small = max(ax, ay), min(ax, ay)
    if big == 0.0:
        return 0.0
    r = small / big
    return big * math.sqrt(fma(r, r, 1.0))


def test_complex_abs_is_numpys():
    rng = np.random.default_rng(1)
    n = 4000
    z = (rng.normal(size=n) * np.exp(rng.uniform(-30, 5, size=n))
         + 1j * rng.normal(size=n) * np.exp(rng.uniform(-30, 5, size=n)))
    z[:4] = [0, 1j, 3 + 3j, -2.5]
    a = np.abs(z)
    for i in range(n):
        assert numpy_cabs(complex(z[i])) == a[i], (i, z[i])


def pw(x):
    n = len(x)
    if n < 8:
        r = 0.0
        for v in x:
            r = r + v
        return r
    if n <= 128:
        r = list(x[:8])
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] = r[j] + x[i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res = res + x[i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pw(x[:n2]) + pw(x[n2:])


@pytest.mark.parametrize("D", [3, 7, 9, 12, 15])
def test_pairwise_sum_tree(D):
    rng = np.random.default_rng(D)
    x = rng.random(1 << D) ** 5
    xs = [float(v) for v in x]
    assert pw(xs) == np.sum(x)
    # the leaves-of-128 + pairwise-tree evaluation the kernel uses
    if D >= 7:
        leaves = [pw(xs[i:i + 128]) for i in range(0, len(xs), 128)]
        assert pairwise_combine(leaves) == np.sum(x)
    # ranges of 2^k processes combine as a pairwise tree too
    if D >= 10:
        for world in (2, 4, 8):
            m = len(xs) // world
            assert pairwise_combine([pw(xs[j * m:(j + 1) * m]) for j in range(world)]) == np.sum(x)


def exact_cumsum_by_chunks(q, B):
    """cdf.cu's walk restated: per chunk, integer ulp increments when the
    chunk stays in one binade of the running sum, else element by element."""
    tot = [math.fsum(q[k:k + B]) for k in range(0, len(q), B)]
    cstart = np.cumsum([0.0] + tot[:-1])
    ends = []
    c = 0.0
    fast = 0
    for k in range(len(tot)):
        lo, hi = k * B, min(len(q), (k + 1) * B)
        done = False
        c0, c1 = cstart[k], cstart[k] + tot[k]
        if c0 >= 2.0 ** -1000 and c > 0.0 and math.frexp(c0)[1] == math.frexp(c1)[1]:
            e = math.frexp(c0)[1] - 1  # c0 in [2^e, 2^(e+1))
            incs = {}
            for p in (0, 1):
                par, tot_inc = p, 0
                for v in q[lo:hi]:
                    f = math.ldexp(v, 52 - e)
                    kk = math.floor(f)
                    fr = f - kk
                    inc = kk + (1 if fr > 0.5 else ((par + kk) & 1 if fr == 0.5 else 0))
                    tot_inc += inc
                    par = (par + inc) & 1
                incs[p] = tot_inc
            if math.frexp(c)[1] - 1 == e:
                m = int(math.ldexp(c, 52 - e))
                me = m + incs[m & 1]
                if me < 2 ** 53:
                    c = math.ldexp(me, e - 52)
                    done = True
                    fast += 1
        if not done:
            for v in q[lo:hi]:
                c = c + v
        ends.append(c)
    return ends, fast


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_exact_cumsum_walk(seed):
    rng = np.random.default_rng(seed)
    n, B = 1 << 14, 64
    p = rng.random(n) ** 8
    p[rng.integers(0, n, 50)] = 0.0
    # ties: values that are exactly half an ulp of typical running sums
    for i in rng.integers(n // 4, n, 40):
        p[i] = math.ldexp(1.0, -60)
    q = p / np.sum(p)
    cdf = np.cumsum(q)
    ends, fast = exact_cumsum_by_chunks([float(v) for v in q], B)
    want = [cdf[min(n, (k + 1) * B) - 1] for k in range(len(ends))]
    assert ends == want
    assert fast > len(ends) // 2  # most chunks take the integer path
