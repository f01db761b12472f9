"""Host logic of the peer-memory remap (comm.swap_args), emulated on CPU.

For every process of a world of 2, 4 or 8, the arguments that
svb_peer_swap_bulk would receive are replayed in numpy with the kernel's
element enumeration (csrc/peer.cu): pairs k in [first, first+count) of the
local region sel_local and the partner's region sel_remote are swapped.
Whole exchanges and every chunk of a chunked one must (a) swap each pair
exactly once and (b) leave the concatenated state equal to the global
device-bit <-> local-bit swap of the reference remap (executor.py:224-281).
"""

import numpy as np
import pytest
import torch

from paper_2509_14098_b200 import comm

BASE = 1000  # fake peer "pointers": rank + BASE


class _State:
    def __init__(self, rows, L):
        self.rows, self.L = rows, L
        self.buf = torch.zeros(rows << L, dtype=torch.complex128)


class _Ctx:
    def __init__(self, world):
        self.peers = {r: BASE + r for r in range(world)}


def _addr(k, rows_bits_L, lbits, sel):
    L = rows_bits_L
    mm = len(lbits)
    free = [b for b in range(L) if b not in lbits]
    selmask = 0
    for i, b in enumerate(lbits):
        if (sel >> (mm - 1 - i)) & 1:
            selmask |= 1 << b
    row = k >> (L - mm)
    e = k & ((1 << (L - mm)) - 1)
    loc = np.full_like(k, selmask)
    for i, b in enumerate(free):
        loc |= ((e >> i) & 1) << b
    return (row << L) | loc


def _replay(states, world, remote, cbits, cval, touched):
    """Apply every process's swap for one (chunk of an) exchange."""
    calls = []
    for w in range(world):
        fake = _State(ROWS, L_)
        args, partners, (keep, ptrs) = comm.swap_args(fake, remote, w, _Ctx(world), cbits, cval)
        lbits, sel_l, sel_r, first, count = keep
        for j in range(len(partners)):
            p = int(ptrs[j]) - BASE
            assert p == partners[j]
            calls.append((w, p, [int(b) for b in lbits], int(sel_l[j]), int(sel_r[j]), int(first[j]),
                          int(count[j])))
    for w, p, lbits, sl, sr, f, c in calls:
        k = np.arange(f, f + c, dtype=np.int64)
        a = _addr(k, L_, lbits, sl)
        b = _addr(k, L_, lbits, sr)
        for x in a:
            touched[w][x] += 1
        for x in b:
            touched[p][x] += 1
        tmp = states[w][a].copy()
        states[w][a] = states[p][b]
        states[p][b] = tmp


L_ = 6
ROWS = 1


@pytest.mark.parametrize("world,remote,cbits", [
    (2, [(0, 5)], None),
    (2, [(0, 0)], None),
    (2, [(0, 3)], [5, 1]),
    (4, [(0, 2), (1, 4)], None),
    (4, [(1, 5), (0, 4)], [0]),
    (8, [(0, 1), (1, 3), (2, 5)], None),
    (8, [(2, 5), (1, 4), (0, 3)], [0, 1]),
])
def test_peer_swap_schedule(world, remote, cbits):
    rng = np.random.default_rng(3)
    n = ROWS << L_
    full = rng.normal(size=world * n) + 1j * rng.normal(size=world * n)
    states = [full[w * n:(w + 1) * n].copy() for w in range(world)]
    touched = [np.zeros(n, dtype=np.int64) for _ in range(world)]
    for cval in range(1 << len(cbits or [])):
        _replay(states, world, remote, cbits, cval, touched)
    # every exchanged amplitude is written exactly once, the rest never
    m = len(remote)
    for w in range(world):
        alpha = 0
        for e, _ in remote:
            alpha = (alpha << 1) | ((w >> e) & 1)
        idx = np.arange(n)
        sel = np.zeros(n, dtype=np.int64)
        for e, lb in remote:
            sel = (sel << 1) | ((idx >> lb) & 1)
        moved = sel != alpha
        assert np.all(touched[w][moved] == 1)
        assert np.all(touched[w][~moved] == 0)
    got = np.concatenate(states)
    nb = (world.bit_length() - 1) + L_
    x = full.reshape((2,) * nb)
    for e, lb in remote:
        x = np.swapaxes(x, nb - 1 - (L_ + e), nb - 1 - lb)
    np.testing.assert_array_equal(got, np.ascontiguousarray(x).reshape(-1))
    assert m >= 1


def test_partner_rounds_are_matchings():
    """Partner j of every process, ordered by sel ^ alpha, pairs processes
    perfectly: in round j each process is the round-j partner of its partner."""
    for world, remote in ((4, [(0, 2), (1, 4)]), (8, [(0, 1), (1, 3), (2, 5)])):
        order = {}
        for w in range(world):
            _, partners, _ = comm.swap_args(_State(ROWS, L_), remote, w, _Ctx(world))
            order[w] = partners
        for j in range(world - 1):
            for w in range(world):
                assert order[order[w][j]][j] == w
