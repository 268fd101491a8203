"""Cold first re-plan of a fresh planner (host preparation stages via
LIVEPUT_TRACE_PREPARE), N=32 known-answer sequence at 1e4 and the bench shape."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import north_star_nseq
from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b
from paper_2403_14097_b200.planner import Planner, reactive_plan
torch.cuda.init()
N32 = [32, 28, 28, 26, 29, 26, 26, 21, 23, 23, 21, 25, 22]
w = lm_1p5b()
for name, ns, trials in [("n32", N32, 10_000), ("n32-again", N32, 10_000), ("bench", north_star_nseq(256, 24), 1_000_000)]:
    t = time.perf_counter()
    p = Planner(w, CostTable(), PlannerOptions(mc_trials=trials))
    t1 = time.perf_counter()
    for i in range(3):
        t2 = time.perf_counter()
        p.dp_optimize(reactive_plan(ns[0], w), ns)
        s = p.stats()
        print(f"{name}: create {1e3*(t1-t):.2f} ms, re-plan {i}: wall {1e3*(time.perf_counter()-t2):.3f} ms, "
              f"prepare {s.prepare_ms:.3f} ms, device {s.total_ms:.3f} ms", file=sys.stderr, flush=True)
    p.close()
