"""Generate tests/golden/plans_1e6.json: the plans of the benchmarked configs at
the sample count they are timed at (1e6 per (n, k) point).

The reference's own tests never reach the Planner's Monte-Carlo branch
(optimizer.cpp:86-90), so these fixtures pin it:

  * 1e6 plans come from the C restatement (oracle/liveput_oracle.c, cache-free,
    multi-threaded).  The compiled reference would need ~1 h per N=256 re-plan
    at 1e6.
  * the restatement itself is cross-checked here against the UNMODIFIED
    reference's Planner::dp_optimize (oracle/_ref) at 1e5 on two bench-shaped
    re-plans (N=256 I=12 GPT-2 and N=128 I=12 GPT-3); those reference plans are
    stored too, so the 1e6 fixtures rest on the reference, not only on the
    restatement.

Cases:
  bench      north_star_nseq(256, 24): bench.py's workload (BASELINE configs[3])
  ns12       north_star_nseq(256, 12): the north-star re-plan
  predict    tools/prof_replan.py PREDICT: forecast-like drops, k <= 8
  config3    the first 60 Proactive(12, arima) re-plans of config 3 (GPT-3 6.7B,
             N=128, tools/data/trace_gen_synthetic_128.json), forecasts from the
             reference's predict(); `current` = adjust_config of the previous plan
  ref_1e5_*  reference dp_optimize at 1e5 (and the restatement's plan, asserted equal)

Run in the dev container (needs /root/reference for the reference legs):
    python tests/golden/make_plans_1e6.py [--only bench,ns12,...]
Floats are float.hex() strings: the GPU test compares them bit for bit.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

from bench import north_star_nseq  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b, lm_6p7b  # noqa: E402

OUT = Path(__file__).resolve().parent / "plans_1e6.json"
PREDICT = [256, 250, 252, 245, 245, 248, 240, 236, 238, 232, 232, 229, 226]
PROFILES = {"lm_1p5b": lm_1p5b, "lm_6p7b": lm_6p7b}


def enc_cfg(c):
    return None if c is None else [c.pipelines, c.stages]


def enc_plan(plan):
    return [[enc_cfg(s.config), s.expected_committed.hex(), s.expected_mig_cost_s.hex()] for s in plan]


def one(name, profile, trials, n_seq, current=None, threads=8):
    w = PROFILES[profile]()
    cur = current if current is not None else O.oracle_reactive(w, n_seq[0])
    t = time.perf_counter()
    plan, fv = O.OraclePlanner(w, CostTable(), PlannerOptions(mc_trials=trials), threads=threads).dp_optimize(
        cur, n_seq, with_value=True)
    dt = time.perf_counter() - t
    print(f"{name}: oracle {dt:.1f} s", flush=True)
    return {"profile": profile, "trials": trials, "current": enc_cfg(cur), "n_seq": list(n_seq),
            "plan": enc_plan(plan), "final_value": fv.hex(), "oracle_s": round(dt, 1)}


def config3(trials, intervals=60):
    import replay as R
    from paper_2403_14097_b200.planner import ForecastConfig
    counts = json.loads(R.TRACE.read_text())["counts"]
    w = lm_6p7b()
    H = I = R.LOOKAHEAD
    fc = ForecastConfig(history_len=H, lookahead=I, capacity=128)
    pw, keep = w.to_c()
    depth_ok = lambda s: bool(O.oracle_lib().or_depth_feasible(pw, s))
    op = O.OraclePlanner(w, CostTable(), PlannerOptions(mc_trials=trials), threads=8)
    replans = []
    cfg, planned = O.oracle_reactive(w, counts[0]), None
    t0 = time.perf_counter()
    for i in range(intervals):
        n = counts[i]
        if i > 0:
            cfg = R.adjust_config(planned, n, depth_ok)
        ns = [n] + O.ref_predict(R.padded_history(counts, i, H), fc, 0)
        plan = op.dp_optimize(cfg, ns)
        planned = plan[0].config
        replans.append({"current": enc_cfg(cfg), "n_seq": ns, "plan": enc_plan(plan)})
        if i % 10 == 9:
            print(f"config3: {i + 1} re-plans, {time.perf_counter() - t0:.0f} s", flush=True)
    return {"profile": "lm_6p7b", "trials": trials, "trace": "tools/data/trace_gen_synthetic_128.json",
            "policy": "Proactive(12, arima, 12)", "replans": replans}


def ref_case(name, profile, trials, n_seq):
    """The unmodified reference's dp_optimize, cross-checked against the restatement."""
    w = PROFILES[profile]()
    cur = O.oracle_reactive(w, n_seq[0])
    t = time.perf_counter()
    ref = O.RefPlanner(w, CostTable(), PlannerOptions(mc_trials=trials)).dp_optimize(cur, n_seq)
    dt = time.perf_counter() - t
    orc = one(name, profile, trials, n_seq, cur)
    assert enc_plan(ref) == orc["plan"], f"{name}: restatement differs from the reference"
    print(f"{name}: reference {dt:.1f} s, restatement identical", flush=True)
    orc["reference_s"] = round(dt, 1)
    orc["reference_plan_equal"] = True
    return orc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    only = set(x for x in a.only.split(",") if x)
    jobs = {
        "bench": lambda: one("bench", "lm_1p5b", 1_000_000, north_star_nseq(256, 24)),
        "ns12": lambda: one("ns12", "lm_1p5b", 1_000_000, north_star_nseq(256, 12)),
        "predict": lambda: one("predict", "lm_1p5b", 1_000_000, PREDICT),
        "config3": lambda: config3(1_000_000),
        "ref_1e5_gpt3_128": lambda: ref_case("ref_1e5_gpt3_128", "lm_6p7b", 100_000,
                                             json.loads((ROOT / "tools/data/trace_gen_synthetic_128.json")
                                                        .read_text())["counts"][100:113]),
        "ref_1e5_ns12": lambda: ref_case("ref_1e5_ns12", "lm_1p5b", 100_000, north_star_nseq(256, 12)),
    }
    for k, fn in jobs.items():
        if only and k not in only:
            continue
        data[k] = fn()
        OUT.write_text(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
