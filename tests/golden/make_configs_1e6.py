"""Generate tests/golden/configs_1e6.json: the strategy sequences of BASELINE
configs 2, 3 and 5 at the sample count they are timed at (1e6 per point), from
the C restatement (oracle/liveput_oracle.c, with its opt-in per-(n, k) memo —
the reference's hist_cache_ — which gives identical results).  The
restatement is pinned to the reference by tests/golden/*.json and by the
reference-vs-restatement legs of make_plans_1e6.py.

  config2   ResNet-152 DP table, N=64, five gen_synthetic(s, 64, 60, 30, 25, 1, 8)
            traces, the simulator's Ideal(12) planning loop (simulator.cpp:183-199,
            296-318): target = reactive_plan (i = 0) or adjust_config(planned_next, n),
            n_seq = [n] + the next 12 true counts (the last count past the end)
  config3i  GPT-3 6.7B, N=128, the 1440-interval trace, the same Ideal(12) loop
  config3p  the same trace with Proactive(12, arima): n_seq = [n] + predict() of the
            history left-padded to 12 (the reference's predictor via oracle/_ref)
  sweep     config 5: N in {16..512} x I in {4..32} (tools/sweep.py availability);
            full plans (points already in the file are kept)

Each re-plan stores (current, n_seq, first step); sweep points store the whole plan.
Run in the dev container (the Proactive forecasts need oracle/_ref):
    python tests/golden/make_configs_1e6.py [--only config2,config3i,config3p,sweep]
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

from oracle import oracle as O  # noqa: E402
from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b, lm_6p7b, resnet152_dp  # noqa: E402

OUT = Path(__file__).resolve().parent / "configs_1e6.json"
TRIALS = 1_000_000


def enc_cfg(c):
    return None if c is None else [c.pipelines, c.stages]


def enc_step(s):
    return [enc_cfg(s.config), s.expected_committed.hex(), s.expected_mig_cost_s.hex()]


def sim_loop(w, counts, forecast=None, lookahead=12):
    """The planning decisions of simulator.cpp:119-318 for Ideal / Proactive."""
    import replay as R
    pw, keep = w.to_c()
    depth_ok = lambda s: bool(O.oracle_lib().or_depth_feasible(pw, s))
    op = O.OraclePlanner(w, CostTable(), PlannerOptions(mc_trials=TRIALS), threads=8, cache=True)
    out, planned = [], None
    for i, n in enumerate(counts):
        cfg = O.oracle_reactive(w, n) if i == 0 else R.adjust_config(planned, n, depth_ok)
        if forecast is None:
            ns = [n] + [counts[i + j] if i + j < len(counts) else counts[-1] for j in range(1, lookahead + 1)]
        else:
            ns = [n] + forecast(i)
        plan = op.dp_optimize(cfg, ns)
        planned = plan[0].config
        out.append({"current": enc_cfg(cfg), "n_seq": ns, "first": enc_step(plan[0])})
    return out


def config2():
    data = json.loads((ROOT / "tools" / "data" / "trace_config2_resnet64.json").read_text())
    w = resnet152_dp()
    res = {}
    for s, tr in data["traces"].items():
        t = time.perf_counter()
        res[s] = sim_loop(w, tr)
        print(f"config2 trace {s}: {len(tr)} re-plans, {time.perf_counter() - t:.0f} s", flush=True)
    return {"profile": "resnet152", "trials": TRIALS, "policy": "Ideal(12)", "traces": res}


def config3(proactive):
    import replay as R
    from paper_2403_14097_b200.planner import ForecastConfig
    counts = json.loads(R.TRACE.read_text())["counts"]
    w = lm_6p7b()
    fc = ForecastConfig(history_len=12, lookahead=12, capacity=128)
    fore = (lambda i: O.ref_predict(R.padded_history(counts, i, 12), fc, 0)) if proactive else None
    t = time.perf_counter()
    seq = sim_loop(w, counts, fore)
    print(f"config3 {'proactive' if proactive else 'ideal'}: {len(seq)} re-plans, {time.perf_counter() - t:.0f} s",
          flush=True)
    return {"profile": "lm_6p7b", "trials": TRIALS, "policy": "Proactive(12, arima)" if proactive else "Ideal(12)",
            "trace": "tools/data/trace_gen_synthetic_128.json", "replans": seq}


def sweep(done=()):
    import sweep as SW
    w = lm_1p5b()
    pts = list(done)
    have = {(p["n"], p["I"]) for p in pts}
    for n in SW.NS:
        for I in SW.IS:
            if (n, I) in have:
                continue
            ns = SW.availability(n, I)
            cur = O.oracle_reactive(w, ns[0])
            t = time.perf_counter()
            plan = O.OraclePlanner(w, CostTable(), PlannerOptions(mc_trials=TRIALS), threads=8,
                                   cache=True).dp_optimize(cur, ns)
            pts.append({"n": n, "I": I, "current": enc_cfg(cur), "n_seq": ns, "plan": [enc_step(s) for s in plan]})
            print(f"sweep N={n} I={I}: {time.perf_counter() - t:.1f} s", flush=True)
            OUT.write_text(json.dumps({**json.loads(OUT.read_text()),
                                       "sweep": {"profile": "lm_1p5b", "trials": TRIALS, "points": pts}},
                                      separators=(",", ":")))
    return {"profile": "lm_1p5b", "trials": TRIALS, "points": pts}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    only = set(x for x in a.only.split(",") if x)
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    jobs = {"config2": config2, "config3i": lambda: config3(False), "config3p": lambda: config3(True),
            "sweep": lambda: sweep(data.get("sweep", {}).get("points", []))}
    for k, fn in jobs.items():
        if only and k not in only:
            continue
        data[k] = fn()
        OUT.write_text(json.dumps(data, separators=(",", ":")))


if __name__ == "__main__":
    main()
