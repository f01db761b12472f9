"""Multi-process remap protocol (comm.exchange) with the gloo backend on CPU.

World sizes 2 and 4; each process holds rows x 2^L amplitudes of a random
global state; after the exchange the concatenated state must equal the
global bit-swap permutation (executor.py:224-281 semantics)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class NumpyMover:
    """CPU twin of CudaMover (same region enumeration as csrc/layout.cu)."""

    def __init__(self, state):
        self.state = state

    def _index(self, lbits, m, sel, off, count):
        L = self.state.L
        free = [b for b in range(L) if b not in lbits]
        selmask = 0
        for i, b in enumerate(lbits):
            if (sel >> (m - 1 - i)) & 1:
                selmask |= 1 << b
        k = np.arange(off, off + count, dtype=np.int64)
        row = k >> (L - m)
        e = k & ((1 << (L - m)) - 1)
        loc = np.full_like(k, selmask)
        for i, b in enumerate(free):
            loc |= ((e >> i) & 1) << b
        return (row << L) | loc

    def pack(self, lbits, m, sel, off, count, out):
        idx = self._index(lbits, m, sel, off, count)
        out[:count] = self.state.buf[torch.from_numpy(idx)]

    def unpack(self, lbits, m, sel, off, count, inp):
        idx = self._index(lbits, m, sel, off, count)
        self.state.buf[torch.from_numpy(idx)] = inp[:count]


class S:
    def __init__(self, buf, rows, L):
        self.buf, self.rows, self.L = buf, rows, L


def _worker(rank, world, port, L, rows, remote, chunk, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_14098_b200 import comm

    rng = np.random.default_rng(7)
    n = rows << L
    full = rng.normal(size=world * n) + 1j * rng.normal(size=world * n)
    st = S(torch.from_numpy(full[rank * n:(rank + 1) * n].copy()), rows, L)
    comm.exchange(st, remote, None, None, mover=NumpyMover(st), chunk_elems=chunk)
    parts = [torch.empty_like(st.buf) for _ in range(world)]
    dist.all_gather(parts, st.buf)
    if rank == 0:
        got = torch.cat(parts).numpy()
        # expected: swap device-id bit e (global bit L+h+e) with local bit lb
        h = rows.bit_length() - 1
        nb = (world.bit_length() - 1) + h + L
        x = full.reshape((2,) * nb)
        for e, lb in remote:
            u = L + h + e
            x = np.swapaxes(x, nb - 1 - u, nb - 1 - lb)
        q.put(float(np.max(np.abs(got - np.ascontiguousarray(x).reshape(-1)))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,rows,L,remote,chunk", [
    (2, 1, 6, [(0, 5)], 7),
    (2, 2, 5, [(0, 0)], 64),
    (4, 1, 6, [(0, 2), (1, 4)], 5),
    (4, 2, 5, [(1, 1), (0, 3)], 1000),
    (8, 1, 6, [(0, 3), (1, 4), (2, 5)], 3),
    (8, 2, 5, [(2, 0), (0, 4), (1, 2)], 1000),
])
def test_exchange_matches_bit_swap(world, rows, L, remote, chunk):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + world * 10 + L + rows
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, rows, remote, chunk, q)) for r in range(world)]
    for p in procs:
        p.start()
    err = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert err == 0.0
