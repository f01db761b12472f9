"""Timeline of one multi-GPU run (SVB200_TRACE=1): sweeps, parts and remap
phases per rank, in ms from the run's first mark.

    SVB200_TRACE=1 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/remap_trace.py qft31_h30-12
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2509_14098_b200 import plan as planmod, run_plan  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
me = dist.get_rank()
plan = planmod.load(str(ROOT / "plans" / f"{sys.argv[1] if len(sys.argv) > 1 else 'qft31_h30-12'}.json.gz"))
for it in range(3):
    res = run_plan(plan)
    torch.cuda.synchronize()
    del res
res = run_plan(plan)
torch.cuda.synchronize()
lines = [f"rank {me}: {lab:32s} {t:9.3f}" for lab, t in res.stats.trace]
out = [None] * dist.get_world_size()
dist.all_gather_object(out, lines)
if me == 0:
    for r, ls in enumerate(out):
        print("\n".join(ls), flush=True)
dist.destroy_process_group()
