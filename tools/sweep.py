"""BASELINE config 5: re-plan latency sweep, N in {16..512} x lookahead I in
{4..32}, GPT-2 1.5B table.

  python tools/sweep.py gpu  --trials 1000000 --out gpurun_out/sweep_gpu.json
  python tools/sweep.py gpu  --trials 1000    --out gpurun_out/sweep_gpu_1e3.json
  python tools/sweep.py cpu  --trials 1000    --out profiles/sweep_ref_1e3.json   (reference, 1 thread)

The availability sequence for (N, I) is a deterministic random walk (drops up
to N/8, gains up to N/16, floor N/2) from a splitmix stream, so every tool and
box sees the same inputs.  `compare` checks GPU and reference plans at the same
trial count are identical.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

NS = [16, 32, 64, 128, 256, 512]
IS = [4, 8, 12, 16, 24, 32]


def _mix(a, b):
    m = (1 << 64) - 1
    z = (a + 0x9E3779B97F4A7C15 * (b + 1)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def availability(n, horizon, seed=2024):
    seq = [n]
    for j in range(horizon):
        r = _mix(seed * 1000003 + n, j)
        if r % 3 == 0:
            step = 1 + (r >> 8) % max(1, n // 8)
            v = max(n // 2, seq[-1] - step)
        elif r % 3 == 1:
            step = (r >> 8) % max(1, n // 16 + 1)
            v = min(n, seq[-1] + step)
        else:
            v = seq[-1]
        seq.append(v)
    return seq


def run_gpu(trials, reps):
    from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b
    from paper_2403_14097_b200.planner import Planner, reactive_plan
    w = lm_1p5b()
    p = Planner(w, CostTable(), PlannerOptions(mc_trials=trials))
    out = []
    for n in NS:
        for I in IS:
            ns = availability(n, I)
            cur = reactive_plan(ns[0], w)
            p.prepare(cur, ns)
            p.execute()  # warm-up (module load, allocations)
            dev = []
            for _ in range(reps):
                p.execute()
                dev.append(p.stats().total_ms)
            e2e = []
            for _ in range(reps):
                t = time.perf_counter()
                plan = p.dp_optimize(cur, ns)
                e2e.append(1e3 * (time.perf_counter() - t))
            st = p.stats()
            out.append({"n": n, "I": I, "n_seq": ns, "trials": trials, "device_ms": min(dev), "e2e_ms": min(e2e),
                        "resolutions": st.resolutions, "mc_pairs": st.mc_pairs,
                        "plan": [[s.config.pipelines, s.config.stages] if s.config else None for s in plan],
                        "values": [[s.expected_committed.hex(), s.expected_mig_cost_s.hex()] for s in plan]})
            print(json.dumps({k: out[-1][k] for k in ("n", "I", "device_ms", "e2e_ms", "resolutions")}), flush=True)
    p.close()
    return out


def run_cpu(trials, max_s):
    import ctypes as C
    from oracle.oracle import RefPlanner, ref_lib
    from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b
    from oracle.oracle import oracle_reactive
    L = ref_lib()
    w = lm_1p5b()
    out = []
    skip_n = set()
    for n in NS:
        for I in IS:
            ns = availability(n, I)
            cur = oracle_reactive(w, ns[0])
            if n in skip_n:
                out.append({"n": n, "I": I, "n_seq": ns, "trials": trials, "ref_ms": None, "skipped": True})
                continue
            rp = RefPlanner(w, CostTable(), PlannerOptions(mc_trials=trials))
            t = time.perf_counter()
            plan = rp.dp_optimize(cur, ns)
            ms = 1e3 * (time.perf_counter() - t)
            out.append({"n": n, "I": I, "n_seq": ns, "trials": trials, "ref_ms": ms,
                        "plan": [[s.config.pipelines, s.config.stages] if s.config else None for s in plan],
                        "values": [[s.expected_committed.hex(), s.expected_mig_cost_s.hex()] for s in plan]})
            print(json.dumps({k: out[-1][k] for k in ("n", "I", "ref_ms")}), flush=True)
            if ms > max_s * 1e3:
                skip_n.add(n)
    return out


def summary(g6_path, g3_path, ref_path, md_path):
    """Rewrite the table of profiles/sweep_summary.md from the three sweep files."""
    g6 = {(r["n"], r["I"]): r for r in json.loads(Path(g6_path).read_text())}
    g3 = {(r["n"], r["I"]): r for r in json.loads(Path(g3_path).read_text())}
    rf = {(r["n"], r["I"]): r for r in json.loads(Path(ref_path).read_text())}
    rows = ["| N | I | MC resolutions (1e6) | GPU (1e6) ms | GPU e2e ms | GPU (1e3) ms | ref (1e3) ms | ref/GPU at 1e3 |",
            "|---|---|---|---|---|---|---|---|"]
    for key in sorted(g6):
        a, b, r = g6[key], g3.get(key, {}), rf.get(key, {})
        ref_ms = r.get("ref_ms")
        ratio = f"{ref_ms / b['device_ms']:.0f}×" if ref_ms and b.get("device_ms") else "—"
        ref_s = f"{ref_ms:.0f}" if ref_ms else "skipped"
        rows.append(f"| {key[0]} | {key[1]} | {a['resolutions']:.3g} | {a['device_ms']:.2f} | {a['e2e_ms']:.2f} | "
                    f"{b.get('device_ms', float('nan')):.2f} | {ref_s} | {ratio} |")
    md = Path(md_path).read_text().splitlines()
    start = next(i for i, l in enumerate(md) if l.startswith("| N | I |"))
    end = start
    while end < len(md) and md[end].startswith("|"):
        end += 1
    Path(md_path).write_text("\n".join(md[:start] + rows + md[end:]) + "\n")


def compare(a_path, b_path):
    a = {(r["n"], r["I"]): r for r in json.loads(Path(a_path).read_text())}
    b = {(r["n"], r["I"]): r for r in json.loads(Path(b_path).read_text())}
    bad = 0
    for key, ra in a.items():
        rb = b.get(key)
        if not rb or "plan" not in rb or "plan" not in ra:
            continue
        same = ra["plan"] == rb["plan"] and ra["values"] == rb["values"]
        bad += not same
        print(key, "identical" if same else "DIFFERENT")
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["gpu", "cpu", "compare", "summary"])
    ap.add_argument("--trials", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--max-s", type=float, default=60.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("files", nargs="*")
    a = ap.parse_args()
    if a.mode == "compare":
        sys.exit(1 if compare(*a.files) else 0)
    if a.mode == "summary":  # gpu_1e6.json gpu_1e3.json ref_1e3.json summary.md
        return summary(*a.files)
    res = run_gpu(a.trials, a.reps) if a.mode == "gpu" else run_cpu(a.trials, a.max_s)
    if a.out:
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text(json.dumps(res))


if __name__ == "__main__":
    main()
