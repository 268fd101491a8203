"""BASELINE config 1: GPT-2 1.5B table (lm_1p5b, P >= 7), N=32, 1e4 samples/point,
forecast-driven planning.  Two trace families, s = 1..5:
  high availability  episodic_trace(s, 32, 60, 9, 8, 16)  (reference test fixture)
  low availability   gen_synthetic(s, 32, 60, 9, 8, 1, 4)
Each trace runs the whole simulator with Proactive(12): ARIMA forecasts feed
dp_optimize every interval, starting from reactive_plan(32) = (4, 8).

  python tools/config1.py gen                        # -> tools/data/trace_config1_gpt2_32.json (needs /root/reference)
  python tools/config1.py gpu --out gpurun_out/config1_gpu_1e4.json
  python tools/config1.py ref --out profiles/config1_ref_1e4.json
  python tools/config1.py compare A.json B.json
"""
import argparse
import json
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
TRACES = ROOT / "tools" / "data" / "trace_config1_gpt2_32.json"


def gen():
    from oracle import oracle as O
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "episodic"], check=True)
    seeds = [str(s) for s in range(1, 6)]
    out = subprocess.run([str(ROOT / "oracle" / "_ref" / "gen_episodic"), "32", "60", "9", "8", "16", *seeds],
                         check=True, capture_output=True, text=True).stdout
    traces = {f"high-{s}": tr for s, tr in json.loads(out).items()}
    for s in range(1, 6):
        traces[f"low-{s}"] = O.ref_gen_synthetic(s, 32, 60, 9, 8, 1, 4)
    TRACES.write_text(json.dumps({"capacity": 32, "interval_s": 60.0, "traces": traces,
                                  "source": "episodic_trace(s,32,60,9,8,16) / gen_synthetic(s,32,60,9,8,1,4)"}))
    print(f"wrote {len(traces)} traces to {TRACES}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["gen", "gpu", "ref", "compare"])
    ap.add_argument("--trials", type=int, default=10_000)
    ap.add_argument("--policy", default="proactive")
    ap.add_argument("--out", default=None)
    ap.add_argument("files", nargs="*")
    a = ap.parse_args()
    if a.mode == "gen":
        return gen()
    if a.mode == "compare":
        x = json.loads(Path(a.files[0]).read_text())["runs"]
        y = json.loads(Path(a.files[1]).read_text())["runs"]
        same = all(x[s]["report"] == y[s]["report"] and x[s]["intervals"] == y[s]["intervals"] for s in x)
        print(f"{len(x)} traces: reports {'identical' if same else 'DIFFERENT'}")
        sys.exit(0 if same else 1)
    from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b
    from paper_2403_14097_b200.planner import policy, simulate
    data = json.loads(TRACES.read_text())
    w = lm_1p5b()
    opt = PlannerOptions(mc_trials=a.trials)
    pol = policy(a.policy)
    runs, times = {}, {}
    if a.mode == "gpu":  # untimed: CUDA context, module loading, first allocations
        simulate(next(iter(data["traces"].values())), w, pol, 1, opt, CostTable(), 60.0, data["capacity"])
    for name, tr in data["traces"].items():
        seed = int(name.split("-")[1])
        t0 = time.perf_counter()
        if a.mode == "gpu":
            rep, ivs = simulate(tr, w, pol, seed, opt, CostTable(), 60.0, data["capacity"])
        else:
            from oracle import oracle as O
            rep, ivs = O.ref_simulate(tr, w, pol, seed, opt, CostTable(), 60.0, data["capacity"])
        times[name] = time.perf_counter() - t0
        runs[name] = {"report": rep, "intervals": ivs}
        print(json.dumps({"trace": name, "seconds": round(times[name], 4), "committed": rep["committed_samples"],
                          "rollbacks": rep["rollback_events"], "suspended": rep["suspended_intervals"]}), flush=True)
    res = {"mode": a.mode, "policy": a.policy, "trials": a.trials, "seconds": times, "runs": runs}
    if a.out:
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text(json.dumps(res))


if __name__ == "__main__":
    main()
