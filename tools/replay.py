"""BASELINE config 3: GPT-3 6.7B (D,P) table, N=128, 1e6 samples/point, the
strategy-sequence replay of a synthetic 24 h trace (1440 one-minute intervals).

Two planning loops of the reference simulator (simulator.cpp:185-199, 296-318):
  --policy ideal      Ideal(12): at interval i the planner sees the true next 12
                      availability counts; `current` is the previous plan's first
                      step (it always fits, so adjust_config leaves it unchanged).
  --policy proactive  Proactive(12, arima, 12): n_seq = [n_i] + predict(history)
                      and `current` = adjust_config(previous plan's first step,
                      n_i).  On the GPU every interval's forecast comes from ONE
                      lp_predict_windows launch over the trace (the history never
                      depends on the decisions), included in the timed total.  One Planner persists across the replay,
as in the CLI (commands.cpp:215-216), so ensembles seen before come from the
histogram cache — the reference's hist_cache_ — on the GPU too.

  python tools/replay.py gpu --trials 1000000 --out gpurun_out/replay_gpu.json
  python tools/replay.py ref --trials 1000 --intervals 240 --out profiles/replay_ref_1e3.json
  python tools/replay.py compare A.json B.json
The trace is tools/data/trace_gen_synthetic_128.json, made by the reference's
gen_synthetic(seed=1, 128, 1440, 216, 200, 1, 8) (trace.cpp:80-180) with
`python tools/replay.py trace` in the dev container.
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
TRACE = ROOT / "tools" / "data" / "trace_gen_synthetic_128.json"
LOOKAHEAD = 12


def make_trace():
    import ctypes as C
    from oracle.oracle import ref_lib
    L = ref_lib()
    buf = (C.c_int * 2000)()
    ln = L.ref_gen_synthetic(1, 128, 1440, 216, 200, 1, 8, buf, 2000)
    counts = list(buf[:ln])
    TRACE.parent.mkdir(parents=True, exist_ok=True)
    TRACE.write_text(json.dumps({"generator": "spotsim::gen_synthetic(1, 128, 1440, 216, 200, 1, 8)",
                                 "interval_s": 60, "counts": counts}))
    print(len(counts), min(counts), max(counts))


def loop(plan_fn, reactive_fn, counts, intervals):
    cur = reactive_fn(counts[0])
    seq, times = [], []
    last = min(intervals, len(counts) - LOOKAHEAD)
    for i in range(last):
        ns = counts[i:i + LOOKAHEAD + 1]
        t = time.perf_counter()
        plan = plan_fn(cur, ns)
        times.append(time.perf_counter() - t)
        nxt = plan[0].config
        seq.append([[nxt.pipelines, nxt.stages] if nxt else None, plan[0].expected_committed.hex(),
                     plan[0].expected_mig_cost_s.hex()])
        cur = nxt
    return seq, times


def adjust_config(planned, n, depth_ok):
    """simulator.cpp:31-43."""
    if planned is not None:
        if n >= planned.pipelines * planned.stages:
            return planned
        d = n // planned.stages
        if d >= 1:
            return type(planned)(d, planned.stages)
    for p in range(n, 0, -1):
        if depth_ok(p):
            return type(planned)(1, p) if planned is not None else _cfg(1, p)
    return None


def _cfg(d, p):
    from paper_2403_14097_b200.model import ParallelConfig
    return ParallelConfig(d, p)


def padded_history(counts, i, H):
    """History at interval i (counts[0..i]) left-padded with its first value to H
    entries, as simulator.cpp:311-313 does before predict()."""
    h = counts[: i + 1]
    return [h[0]] * max(0, H - len(h)) + h


def loop_proactive(plan_fn, reactive_fn, forecast_fn, depth_ok, counts, intervals):
    seq, times = [], []
    last = min(intervals, len(counts))
    cfg, planned = reactive_fn(counts[0]), None
    for i in range(last):
        n = counts[i]
        if i > 0:
            cfg = adjust_config(planned, n, depth_ok)
        ns = [n] + forecast_fn(i)
        t = time.perf_counter()
        plan = plan_fn(cfg, ns)
        times.append(time.perf_counter() - t)
        planned = plan[0].config
        seq.append([[planned.pipelines, planned.stages] if planned else None, plan[0].expected_committed.hex(),
                    plan[0].expected_mig_cost_s.hex(), ns[1:]])
    return seq, times


def simulate_mode(a):
    """The whole simulator run() (simulator.cpp:119-340) of config 3: the
    ledger, rollbacks and sample accounting around 1440 re-plans, on this
    library (lp_simulate) or the reference (oracle/_ref), seed 1."""
    if a.mode == "sim-compare":
        x = json.loads(Path(a.files[0]).read_text())
        y = json.loads(Path(a.files[1]).read_text())
        same = x["report"] == y["report"] and x["intervals"] == y["intervals"]
        print(f"reports {'identical' if same else 'DIFFERENT'} ({len(x['intervals'])} intervals)")
        sys.exit(0 if same else 1)
    counts = json.loads(TRACE.read_text())["counts"][: a.intervals]
    from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_6p7b
    from paper_2403_14097_b200.planner import policy, simulate
    w = lm_6p7b()
    opt = PlannerOptions(mc_trials=a.trials)
    pol = policy(a.policy)
    if a.mode == "sim-gpu":  # untimed: CUDA context, module loading (a short prefix at 1e3)
        simulate(counts[:40], w, pol, 1, PlannerOptions(mc_trials=1000), CostTable(), 60.0, 128)
    t0 = time.perf_counter()
    if a.mode == "sim-gpu" and a.seeds > 1:
        from paper_2403_14097_b200.planner import simulate_batch
        runs = simulate_batch(counts, w, pol, list(range(1, a.seeds + 1)), opt, CostTable(), 60.0, 128)
        total = time.perf_counter() - t0
        print(json.dumps({"mode": a.mode, "policy": a.policy, "trials": a.trials, "seeds": a.seeds, "total_s": total,
                          "committed_samples": [r[0]["committed_samples"] for r in runs]}))
        return
    if a.mode == "sim-gpu":
        rep, ivs = simulate(counts, w, pol, 1, opt, CostTable(), 60.0, 128)
    else:
        from oracle import oracle as O
        rep, ivs = O.ref_simulate(counts, w, pol, 1, opt, CostTable(), 60.0, 128)
    total = time.perf_counter() - t0
    res = {"mode": a.mode, "policy": a.policy, "trials": a.trials, "intervals": len(ivs), "total_s": total,
           "report": rep, "intervals": ivs}
    print(json.dumps({k: v for k, v in res.items() if k not in ("report", "intervals")} |
                     {"committed_samples": rep["committed_samples"], "rollback_events": rep["rollback_events"]}))
    if a.out:
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text(json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["trace", "gpu", "ref", "compare", "sim-gpu", "sim-ref", "sim-compare"])
    ap.add_argument("--trials", type=int, default=1_000_000)
    ap.add_argument("--intervals", type=int, default=1440)
    ap.add_argument("--no-cache", action="store_true")
    ap.add_argument("--policy", choices=["ideal", "proactive", "reactive", "checkpoint", "redundancy"], default="ideal")
    ap.add_argument("--seeds", type=int, default=1, help="sim-gpu: seeds 1..S in one lp_simulate_batch")
    ap.add_argument("--out", default=None)
    ap.add_argument("files", nargs="*")
    a = ap.parse_args()
    if a.mode == "trace":
        return make_trace()
    if a.mode.startswith("sim"):
        return simulate_mode(a)
    if a.mode == "compare":
        x = json.loads(Path(a.files[0]).read_text())["sequence"]
        y = json.loads(Path(a.files[1]).read_text())["sequence"]
        m = min(len(x), len(y))
        same = x[:m] == y[:m]
        print(f"compared {m} intervals: {'identical' if same else 'DIFFERENT'}")
        sys.exit(0 if same else 1)
    counts = json.loads(TRACE.read_text())["counts"]
    from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_6p7b
    w = lm_6p7b()
    opt = PlannerOptions(mc_trials=a.trials)
    H = I = LOOKAHEAD
    if a.mode == "gpu":
        from paper_2403_14097_b200 import _abi
        from paper_2403_14097_b200.planner import ForecastConfig, Planner, predict_windows, reactive_plan
        p = Planner(w, CostTable(), opt)
        if not a.no_cache:
            p.set_hist_cache(True)
        t0 = time.perf_counter()
        if a.policy == "ideal":
            seq, times = loop(p.dp_optimize, lambda n: reactive_plan(n, w), counts, a.intervals)
        else:
            cap = json.loads(TRACE.read_text()).get("capacity", 128)
            # window w of [c0]*(H-1) + counts + I pad values has history padded_history(counts, w, H)
            series = [counts[0]] * (H - 1) + counts + [0] * I
            preds, _ = predict_windows(series, ForecastConfig(history_len=H, lookahead=I, capacity=cap), ["arima"])
            pw, keep = w.to_c()
            depth_ok = lambda s: bool(_abi.lib().lp_depth_feasible(pw, s))
            seq, times = loop_proactive(p.dp_optimize, lambda n: reactive_plan(n, w), lambda i: preds[i][0],
                                        depth_ok, counts, a.intervals)
        total = time.perf_counter() - t0
    else:
        from oracle import oracle as O
        from paper_2403_14097_b200.planner import ForecastConfig
        p = O.RefPlanner(w, CostTable(), opt)
        t0 = time.perf_counter()
        if a.policy == "ideal":
            seq, times = loop(p.dp_optimize, lambda n: O.oracle_reactive(w, n), counts, a.intervals)
        else:
            cap = json.loads(TRACE.read_text()).get("capacity", 128)
            fc = ForecastConfig(history_len=H, lookahead=I, capacity=cap)
            pw, keep = w.to_c()
            depth_ok = lambda s: bool(O.ref_lib().ref_depth_feasible(pw, s))
            seq, times = loop_proactive(p.dp_optimize, lambda n: O.oracle_reactive(w, n),
                                        lambda i: O.ref_predict(padded_history(counts, i, H), fc, 0),
                                        depth_ok, counts, a.intervals)
        total = time.perf_counter() - t0
    res = {"mode": a.mode, "policy": a.policy, "trials": a.trials, "intervals": len(seq), "total_s": total,
           "mean_ms": 1e3 * total / max(1, len(seq)), "max_ms": 1e3 * max(times),
           "first_ms": 1e3 * times[0], "cache": not a.no_cache, "sequence": seq}
    print(json.dumps({k: v for k, v in res.items() if k != "sequence"}), flush=True)
    if a.out:
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text(json.dumps(res))


if __name__ == "__main__":
    main()
