"""BASELINE config 2: ResNet-152 data-parallel table (the synthesised
`resnet152_dp` profile: fits at P=1, so every depth is feasible — the full
space), N=64, high-preemption traces gen_synthetic(s, 64, 60, 30,
25, 1, 8) for s = 1..5 (tools/data/trace_config2_resnet64.json), planned with
Ideal(12) so k is not capped by the forecaster's max_step.  Runs the whole
simulator (lp_simulate) per trace.

  python tools/config2.py gpu --trials 1000000 --out gpurun_out/config2_gpu_1e6.json
  python tools/config2.py gpu --trials 1000 --out gpurun_out/config2_gpu_1e3.json
  python tools/config2.py ref --trials 1000 --out profiles/config2_ref_1e3.json
  python tools/config2.py compare A.json B.json
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
TRACES = ROOT / "tools" / "data" / "trace_config2_resnet64.json"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["gpu", "ref", "compare"])
    ap.add_argument("--trials", type=int, default=1_000_000)
    ap.add_argument("--policy", default="ideal")
    ap.add_argument("--out", default=None)
    ap.add_argument("files", nargs="*")
    a = ap.parse_args()
    if a.mode == "compare":
        x = json.loads(Path(a.files[0]).read_text())["runs"]
        y = json.loads(Path(a.files[1]).read_text())["runs"]
        same = all(x[s]["report"] == y[s]["report"] and x[s]["intervals"] == y[s]["intervals"] for s in x)
        print(f"{len(x)} traces: reports {'identical' if same else 'DIFFERENT'}")
        sys.exit(0 if same else 1)
    from paper_2403_14097_b200.model import CostTable, PlannerOptions, resnet152_dp
    from paper_2403_14097_b200.planner import policy, simulate
    data = json.loads(TRACES.read_text())
    w = resnet152_dp()
    opt = PlannerOptions(mc_trials=a.trials)
    pol = policy(a.policy)
    runs, times = {}, {}
    if a.mode == "gpu":  # untimed: CUDA context, module loading, first allocations
        first = next(iter(data["traces"].values()))
        simulate(first, w, pol, 1, opt, CostTable(), 60.0, data["capacity"])
    for s, tr in data["traces"].items():
        t0 = time.perf_counter()
        if a.mode == "gpu":
            rep, ivs = simulate(tr, w, pol, int(s), opt, CostTable(), 60.0, data["capacity"])
        else:
            from oracle import oracle as O
            rep, ivs = O.ref_simulate(tr, w, pol, int(s), opt, CostTable(), 60.0, data["capacity"])
        times[s] = time.perf_counter() - t0
        runs[s] = {"report": rep, "intervals": ivs}
        print(json.dumps({"trace": s, "seconds": round(times[s], 4), "committed": rep["committed_samples"],
                          "rollbacks": rep["rollback_events"], "suspended": rep["suspended_intervals"]}), flush=True)
    res = {"mode": a.mode, "policy": a.policy, "trials": a.trials, "seconds": times, "runs": runs}
    if a.out:
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text(json.dumps(res))


if __name__ == "__main__":
    main()
