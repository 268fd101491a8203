"""Host-side breakdown of one end-to-end re-plan (bench.py workload):
prepare (host tables + H2D), execute (launches), fetch (sync + D2H)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from bench import north_star_nseq  # noqa: E402


def main():
    import torch
    from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b
    from paper_2403_14097_b200.planner import Planner, reactive_plan
    w = lm_1p5b()
    ns = north_star_nseq(256, 24)
    p = Planner(w, CostTable(), PlannerOptions(mc_trials=1_000_000))
    cur = reactive_plan(ns[0], w)
    for _ in range(3):
        p.dp_optimize(cur, ns)
    tp, te, tf, tt = [], [], [], []
    for _ in range(20):
        t0 = time.perf_counter()
        p.prepare(cur, ns)
        t1 = time.perf_counter()
        p.execute()
        t2 = time.perf_counter()
        p.fetch(len(ns) - 1)
        t3 = time.perf_counter()
        tp.append(t1 - t0); te.append(t2 - t1); tf.append(t3 - t2); tt.append(t3 - t0)
        s = p.stats()
    med = lambda v: sorted(v)[len(v) // 2] * 1e3
    print(f"prepare {med(tp):.3f} ms (lib prepare_ms {s.prepare_ms:.3f}), execute {med(te):.3f} ms, "
          f"fetch {med(tf):.3f} ms, total {med(tt):.3f} ms; device hist {s.hist_ms:.3f} dp {s.dp_ms:.3f}; "
          f"h2d {s.h2d_bytes} B")
    t0 = time.perf_counter()
    for _ in range(20):
        p.dp_optimize(cur, ns)
    print(f"dp_optimize {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
