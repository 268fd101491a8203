"""Per-re-plan timing of the config 2 traces (diagnostic for tools/config2.py):
two passes of the full simulation per trace, then the Ideal(12) planning loop
with the histogram cache on and per-re-plan stats.  Output: profiles/config2_replans_1e6.log"""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2403_14097_b200.model import CostTable, PlannerOptions, resnet152_dp
from paper_2403_14097_b200.planner import Planner, reactive_plan, policy, simulate
from paper_2403_14097_b200.model import PROFILES
trials = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
tfile = sys.argv[2] if len(sys.argv) > 2 else 'trace_config2_resnet64.json'
data = json.load(open(Path(__file__).parent / 'data' / tfile))
w = PROFILES[sys.argv[3]]() if len(sys.argv) > 3 else resnet152_dp()
for rep in range(2):
    for s, tr in data['traces'].items():
        t0 = time.perf_counter()
        simulate(tr, w, policy('ideal'), int(s.split('-')[-1]), PlannerOptions(mc_trials=trials), CostTable(), 60.0, data['capacity'])
        print('sim pass', rep, 'trace', s, round(time.perf_counter() - t0, 4), flush=True)
for s, tr in data['traces'].items():
    p = Planner(w, CostTable(), PlannerOptions(mc_trials=trials, interval_s=60.0))
    p.set_hist_cache(True)
    cur = reactive_plan(tr[0], w)
    rows = []
    for i in range(len(tr) - 1):
        ns = [tr[min(i + j, len(tr) - 1)] for j in range(13)]
        t = time.perf_counter(); plan = p.dp_optimize(cur, ns); dt = time.perf_counter() - t
        st = p.stats()
        rows.append((round(dt * 1e3, 2), i, st.mc_pairs, st.exact_pairs, st.cached_pairs, round(st.hist_ms, 2),
                     round(st.dp_ms, 2), round(st.total_ms, 2), round(st.prepare_ms, 2), ns[:5]))
        nxt = plan[0].config
        cur = nxt if nxt is not None and nxt.pipelines * nxt.stages <= ns[1] else reactive_plan(ns[1], w)
    tot = sum(r[0] for r in rows)
    print('trace', s, 'replans', len(rows), 'sum ms', round(tot, 1), 'median', sorted(r[0] for r in rows)[len(rows) // 2])
    for r in sorted(rows, reverse=True)[:6]: print('  ', r)
