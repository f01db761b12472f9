"""Host-side cost of one run_plan call (enqueue) and of its wait() (event
reads, drift check), against the device time of the circuit: shows whether
back-to-back circuits are host-bound."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2509_14098_b200 import executor, plan as planmod, run_plan  # noqa: E402


def main(name="qft30_h30-12", steps=20):
    plan = planmod.load(str(Path(__file__).resolve().parent.parent / "plans" / f"{name}.json.gz"))
    for _ in range(3):
        run_plan(plan).wait()
    torch.cuda.synchronize()
    for prof in (False, True, False):
        executor.PROFILE_SWEEPS = prof
        enq, wt = [], []
        t0 = time.perf_counter()
        prev = None
        for _ in range(steps):
            a = time.perf_counter()
            r = run_plan(plan, wait=False)
            enq.append(time.perf_counter() - a)
            if prev is not None:
                a = time.perf_counter()
                prev.wait()
                wt.append(time.perf_counter() - a)
            prev = r
        prev.wait()
        torch.cuda.synchronize()
        tot = (time.perf_counter() - t0) / steps
        print(f"{name} profile={prof}: enqueue {1e3 * sum(enq) / len(enq):.3f} ms, wait {1e3 * sum(wt) / len(wt):.3f} ms, "
              f"wall per circuit {1e3 * tot:.3f} ms")
    import cProfile
    import pstats

    executor.PROFILE_SWEEPS = True
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(steps):
        run_plan(plan, wait=False).wait()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main(*sys.argv[1:2])
