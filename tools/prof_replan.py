"""Profiling driver: one prepared re-plan executed --reps times (for ncu /
launch lists).  Cases:
  bench    BASELINE configs[3] (N=256, I=24, 1e6, k up to 40: counter variant)
  predict  N=256, I=12, 1e6, forecast-like drops k <= 8 (register variant)
  n32      N=32, I=12, the known-answer sequence (latency floor; use --trials 10000)
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from bench import north_star_nseq  # noqa: E402

N32 = [32, 28, 28, 26, 29, 26, 26, 21, 23, 23, 21, 25, 22]  # SURVEY §8c known-answer sequence
PREDICT = [256, 250, 252, 245, 245, 248, 240, 236, 238, 232, 232, 229, 226]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="bench", choices=["bench", "predict", "ns12", "n32"])
    ap.add_argument("--trials", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import torch
    from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b
    from paper_2403_14097_b200.planner import Planner, reactive_plan
    w = lm_1p5b()
    ns = {"bench": north_star_nseq(256, 24), "predict": PREDICT, "ns12": north_star_nseq(256, 12), "n32": N32}[a.case]
    p = Planner(w, CostTable(), PlannerOptions(mc_trials=a.trials))
    cur = reactive_plan(ns[0], w)
    p.prepare(cur, ns)
    for _ in range(a.reps):
        t = time.perf_counter()
        p.execute()
        s = p.stats()
        print(f"{a.case}: total {s.total_ms:.3f} ms hist {s.hist_ms:.3f} dp {s.dp_ms:.3f} prep {s.prepare_ms:.3f} "
              f"res {s.resolutions} scen {s.scenarios} launches {s.kernel_launches} "
              f"wall {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
    plan = p.fetch(len(ns) - 1)
    for _ in range(3):  # end to end through lp_replan (host tables + H2D + kernels + D2H)
        t = time.perf_counter()
        p.dp_optimize(cur, ns)
        s = p.stats()
        print(f"{a.case}: e2e {1e3 * (time.perf_counter() - t):.3f} ms (prepare {s.prepare_ms:.3f} ms, "
              f"h2d {s.h2d_bytes} B)", flush=True)
    print([(x.config.pipelines, x.config.stages) if x.config else None for x in plan])
    p.close()


if __name__ == "__main__":
    main()
