"""Plan containers and the JSON wire format (reference plan.py:171-201)."""

import json

from conftest import plan_from_doc
from paper_2509_14098_b200 import plan as planmod


def test_json_round_trip_is_byte_identical(grid_docs):
    for doc in grid_docs[:200]:
        text = json.dumps(doc["plan"], indent=2, sort_keys=True)
        plan = planmod.from_json(text)
        assert planmod.to_json(plan) == text
        assert plan.num_ranks == 1 << plan.g
        assert plan.block_len == 1 << (plan.d - plan.g)


def test_bench_plans_load():
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent / "plans"
    meta = json.loads((root / "plans.json").read_text())
    for name, m in meta.items():
        p = planmod.load(str(root / f"{name}.json.gz"))
        assert p.d == m["d"] and p.g == m["g"]
        assert sum(t.kind == "ApplyFused" for t in p.tasks) == m["apply_fused"]


def test_ghz3_layouts(grid_docs):
    # test_plan.py:23-28 golden
    plan = plan_from_doc(next(d for d in grid_docs if d["name"] == "ghz3-2")["plan"])
    assert plan.layout_phases == [[1, 2, 0], [0, 2, 1]]
    assert [t.kind for t in plan.tasks] == ["Alloc", "ApplyFused", "Pack", "Exchange", "Unpack", "ApplyFused", "Free"]
