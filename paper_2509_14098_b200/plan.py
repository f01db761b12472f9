"""The executor's input contract: an SPMD task list over a qubit layout.

A plan is what the reference's host-side partitioner emits
(``svpart/plan.py:24-46`` ``ExecutionPlan``/``Task``; ``lower`` at
``plan.py:105-168``).  The partitioner runs unchanged on the host; this module
only holds the container types and the JSON wire format
(``plan.py:171-201``), so plans produced by the reference load here without
the reference installed (the GPU box has no copy of it).

Layout conventions (``plan.py:3-8``): ``layout_phases[phase][q]`` is the bit
position of qubit line q counted from the most significant bit of the
storage index; positions ``< g`` select the rank, the rest index the
rank-local block of ``2^(d-g)`` amplitudes.

Any object with the same attribute names (``d, g, layout_phases, tasks`` and
tasks with ``id, kind, deps, payload``) is accepted by the executor, so a
reference ``svpart.plan.ExecutionPlan`` can be passed directly.
"""

from __future__ import annotations

import gzip
import json
from dataclasses import dataclass


@dataclass(frozen=True)
class Task:
    id: int
    kind: str  # Alloc | Pack | Exchange | Unpack | ApplyFused | Free
    deps: tuple[int, ...]
    payload: dict


@dataclass
class ExecutionPlan:
    d: int
    g: int
    layout_phases: list[list[int]]
    tasks: list[Task]
    version: int = 1

    @property
    def num_ranks(self) -> int:
        return 1 << self.g

    @property
    def block_len(self) -> int:
        return 1 << (self.d - self.g)


def to_json(plan) -> str:
    """Same document shape and key order as the reference (sorted keys, indent 2)."""
    doc = {
        "version": getattr(plan, "version", 1),
        "d": plan.d,
        "g": plan.g,
        "layout_phases": [list(p) for p in plan.layout_phases],
        "tasks": [
            {"id": t.id, "kind": t.kind, "deps": list(t.deps), "payload": t.payload}
            for t in plan.tasks
        ],
    }
    return json.dumps(doc, indent=2, sort_keys=True)


def from_json(text: str) -> ExecutionPlan:
    doc = json.loads(text)
    tasks = [
        Task(id=t["id"], kind=t["kind"], deps=tuple(t["deps"]), payload=t["payload"])
        for t in doc["tasks"]
    ]
    return ExecutionPlan(
        d=doc["d"],
        g=doc["g"],
        layout_phases=[list(p) for p in doc["layout_phases"]],
        tasks=tasks,
        version=doc.get("version", 1),
    )


def load(path: str) -> ExecutionPlan:
    """Read a plan JSON file (optionally gzip-compressed)."""
    opener = gzip.open if str(path).endswith(".gz") else open
    with opener(path, "rt") as fh:
        return from_json(fh.read())


def save(plan, path: str) -> None:
    opener = gzip.open if str(path).endswith(".gz") else open
    with opener(path, "wt") as fh:
        fh.write(to_json(plan))
