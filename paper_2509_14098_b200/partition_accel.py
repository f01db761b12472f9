"""Faster drop-ins for the reference partitioner's two hot spots (SURVEY.md
§8(f) row 4), producing byte-identical partition trees.

The reference partitioner (``svpart.partitioner.partition``) runs on the host
before every simulation; for QV-30/34 it takes 10-14 s, longer than the GPU
run.  A profile (round 1, QV-30 [30,12], 13.5 s) shows two costs:

* ``centrality.compute_reach`` (centrality.py:70-89), 9.0 s.  Its min-plus
  rows take 0.25 s; the rest builds a per-node ``rn`` dict of every
  reachable node (O(V^2) Python objects).  The partitioner only reads
  ``table.cc`` (partitioner.py:158), which needs each node's reachable-set
  size and distance sum.  ``closeness`` below computes the same rows and
  derives cc from row counts and sums; ``table.reach`` is rebuilt by the
  reference's own ``compute_reach`` only if a caller reads it.
* ``forward_pass``'s ``absorb_round`` (partitioner.py:165-182), 3.4 s: it
  rescans every gate, calling ``ready`` 1.2M times.  Because a gate's
  predecessors on every line come earlier in ``gate_order``, the first scan
  already absorbs everything absorbable, in ``gate_order`` order; the later
  scans only confirm that nothing else is.  ``forward_pass`` below absorbs
  the same gates in the same order with a min-heap over the frontier.

``install()`` points ``svpart.partitioner`` at these two functions; trees are
checked byte-for-byte against the reference in tests/test_partition_accel.py.
"""

from __future__ import annotations

import heapq
import sys
from collections.abc import Mapping

import numpy as np

_INF = np.int64(2**62)  # centrality.py:22


def _ref(name: str):
    mod = sys.modules.get(name)
    if mod is None:
        import importlib

        mod = importlib.import_module(name)
    return mod


class _LazyReach(Mapping):
    """table.reach on demand: the reference's compute_reach, run on first use."""

    def __init__(self, graph):
        self._graph = graph
        self._table = None

    def _get(self):
        if self._table is None:
            self._table = _ref("svpart.centrality").compute_reach(self._graph)
        return self._table

    def __getitem__(self, k):
        return self._get()[k]

    def __iter__(self):
        return iter(self._get())

    def __len__(self):
        return len(self._graph.nodes)


def reach_counts(graph) -> tuple[list, np.ndarray, np.ndarray]:
    """(topological ids, |RN|, sum of distances) per node.

    The rows restate compute_reach (centrality.py:70-83): in reverse
    topological order a node's row is the elementwise minimum over its
    downstream neighbours u of row(u) + |l_v - l_u|, with the entry of u
    itself set to that edge weight.  Adjacency as centrality.py:55-67.
    """
    C = _ref("svpart.centrality")
    out_id = _ref("svpart.graph").OUTPUT_ID
    nodes = graph.nodes
    nbrs: dict[int, set] = {nid: set() for nid in nodes}
    for dim, (p, c) in graph.edges.items():
        if c == out_id:
            continue
        if nodes[p].l >= nodes[c].l:
            raise C.CycleDetected(f"edge {dim} does not increase l")
        nbrs[p].add(c)
    ids = graph.topo_order()
    index = {nid: i for i, nid in enumerate(ids)}
    v = len(ids)
    # int32 rows when safe: a path has fewer than V edges, each of weight
    # |delta l| <= max l, so with V < 2^15 and max l < 2^15 every distance (and
    # distance + edge) stays below the 2^30 sentinel; otherwise int64 as the reference
    small = v * v < (1 << 30) and max((n.l for n in nodes.values()), default=0) < (1 << 15)
    dt, inf = (np.int32, np.int32(1 << 30)) if small else (np.int64, _INF)
    rows = np.full((v, v), inf, dtype=dt)
    for nid in reversed(ids):
        row = rows[index[nid]]
        lv = nodes[nid].l
        for u in sorted(nbrs[nid]):
            w = abs(nodes[u].l - lv)
            j = index[u]
            cand = np.minimum(rows[j] + dt(w), inf)
            cand[j] = w
            np.minimum(row, cand, out=row)
    hit = rows < inf
    size = hit.sum(axis=1)
    dist = np.where(hit, rows, 0).sum(axis=1, dtype=np.int64)
    return ids, size, dist


def closeness(graph):
    """centrality.closeness (centrality.py:114-126) with cc from row counts."""
    C = _ref("svpart.centrality")
    ids, size, dist = reach_counts(graph)
    n = len(graph.nodes)
    cc = {}
    for i, nid in enumerate(ids):
        s, dsum = int(size[i]), int(dist[i])
        cc[nid] = 0.0 if s == 0 else (s / dsum) * (s / n)
    return C.CentralityTable(reach=_LazyReach(graph), cc=cc, n=n)


def forward_pass(graph, centrality, L, *, candidate_lines=None, level=0):
    """partitioner.forward_pass (partitioner.py:123-228) with an event-driven
    absorb round; same partitions, same gate order, same errors."""
    P = _ref("svpart.partitioner")
    lines = tuple(range(graph.d)) if candidate_lines is None else tuple(sorted(candidate_lines))
    width = min(L, len(lines))
    gate_order = graph.gate_ids()
    nodes = graph.nodes
    per_line: dict[int, list] = {q: [] for q in range(graph.d)}
    for gid in gate_order:
        for q in nodes[gid].qubits:
            per_line[q].append(gid)
    done: set = set()
    head = {q: 0 for q in range(graph.d)}  # first possibly-pending position per line

    def pending(q):
        seq = per_line[q]
        i = head[q]
        while i < len(seq) and seq[i] in done:
            i += 1
        head[q] = i
        return seq[i] if i < len(seq) else None

    def at_frontier(gid):
        return all(pending(q) == gid for q in nodes[gid].qubits)

    def score(q):
        for gid in per_line[q][head[q]:]:
            if gid not in done and not nodes[gid].gate.is_diagonal:
                return centrality.cc[gid]
        return -1.0

    def choose(forced):
        order = sorted((q for q in lines if q not in forced), key=lambda q: (-score(q), q))
        chosen = set(forced)
        for q in order:
            if len(chosen) >= width:
                break
            chosen.add(q)
        return chosen

    def absorb(local):
        taken = []
        heap = sorted({g for g in (pending(q) for q in range(graph.d)) if g is not None and at_frontier(g)})
        queued = set(heap)
        while heap:
            gid = heapq.heappop(heap)
            node = nodes[gid]
            away = {slot for slot, q in enumerate(node.qubits) if q not in local}
            if away and not P.can_pass_through(node.gate, away):
                continue  # stays pending; so do its successors this round
            done.add(gid)
            taken.append(gid)
            for q in node.qubits:
                g = pending(q)
                if g is not None and g not in queued and at_frontier(g):
                    queued.add(g)
                    heapq.heappush(heap, g)
        return taken

    parts = []
    while len(done) < len(gate_order):
        local = choose(set())
        taken = absorb(local)
        if not taken:
            first = next(gid for gid in gate_order if gid not in done)
            node = nodes[first]
            need = P._required_lines(node.gate, node.qubits)
            if not need <= set(lines) or len(need) > width:
                raise P.BudgetTooSmall(
                    f"gate {node.gate.kind} on {node.qubits} needs "
                    f"{sorted(need)} local but budget is {L}"
                )
            local = choose(need)
            taken = absorb(local)
            if not taken:
                raise P.PartitionError("frontier stalled; dependency order broken")
        parts.append(P.Partition(
            level=level,
            local_dims=tuple(sorted(local)),
            global_dims=tuple(q for q in range(graph.d) if q not in local),
            gate_ids=tuple(taken),
            passthrough=frozenset(g for g in taken if any(q not in local for q in nodes[g].qubits)),
        ))
    return parts


_saved: dict = {}


def install() -> None:
    """Route svpart.partitioner.partition through the faster functions."""
    P = _ref("svpart.partitioner")
    if not _saved:
        _saved.update(closeness=P.closeness, forward_pass=P.forward_pass)
    P.closeness = closeness
    P.forward_pass = forward_pass


def uninstall() -> None:
    if _saved:
        P = _ref("svpart.partitioner")
        P.closeness = _saved["closeness"]
        P.forward_pass = _saved["forward_pass"]
