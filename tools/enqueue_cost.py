"""Host cost of enqueueing one prepared re-plan (lp_execute returns after the
launches are queued) against its device time: the case for or against CUDA
graphs.  Cases: the bench re-plan (N=256, I=24, 1e6), the north-star I=12
re-plan, and the N=32 known-answer re-plan at 1e4 (latency floor)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import north_star_nseq
from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b
from paper_2403_14097_b200.planner import Planner, reactive_plan

N32 = [32, 28, 28, 26, 29, 26, 26, 21, 23, 23, 21, 25, 22]
w = lm_1p5b()
for name, ns, trials in [("bench", north_star_nseq(256, 24), 1_000_000), ("ns12", north_star_nseq(256, 12), 1_000_000),
                         ("n32", N32, 10_000)]:
    p = Planner(w, CostTable(), PlannerOptions(mc_trials=trials))
    p.prepare(reactive_plan(ns[0], w), ns)
    enq, dev, launches = [], [], 0
    for i in range(12):
        torch.cuda.synchronize()
        t = time.perf_counter()
        p.execute()
        enq.append((time.perf_counter() - t) * 1e3)
        p.fetch(len(ns) - 1)
        s = p.stats()
        dev.append(s.total_ms)
        launches = s.kernel_launches
    enq, dev = sorted(enq[2:]), sorted(dev[2:])
    print(f"{name}: enqueue median {enq[len(enq)//2]:.3f} ms, device median {dev[len(dev)//2]:.3f} ms, "
          f"kernel launches {launches}")
    p.close()
