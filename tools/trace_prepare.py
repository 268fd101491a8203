import sys, time
sys.path.insert(0, '/root/repo')
from bench import north_star_nseq
from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b
from paper_2403_14097_b200.planner import Planner, reactive_plan
w = lm_1p5b(); ns = north_star_nseq(256, 24)
p = Planner(w, CostTable(), PlannerOptions(mc_trials=1_000_000))
cur = reactive_plan(ns[0], w)
for i in range(6):
    t = time.perf_counter(); p.dp_optimize(cur, ns); dt = time.perf_counter() - t
    s = p.stats()
    print(f"replan {i}: wall {dt*1e3:.3f} ms device {s.total_ms:.3f} prep {s.prepare_ms:.3f}", file=sys.stderr, flush=True)
