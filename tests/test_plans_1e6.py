"""Plans at the sample count the benchmarks are timed at (1e6 per (n, k)).

tests/golden/plans_1e6.json is written by tests/golden/make_plans_1e6.py from
the C restatement (oracle/liveput_oracle.c), which that script cross-checks
against the unmodified reference's Planner::dp_optimize (oracle/_ref) at 1e5
on two bench-shaped re-plans (stored here as ref_1e5_*).  The device plan must
match every step's configuration and both FP64 step values bit for bit
(tolerance 0): optimizer.cpp:140-205 over preemption.cpp:47-59 ensembles.
"""
import pytest

from conftest import load_golden
from paper_2403_14097_b200.model import CostTable, ParallelConfig, PlannerOptions, PROFILES

FIX = load_golden("plans_1e6")


def _cfg(x):
    return None if x is None else ParallelConfig(*x)


def _rows(plan):
    return [[None if s.config is None else [s.config.pipelines, s.config.stages],
             s.expected_committed.hex(), s.expected_mig_cost_s.hex()] for s in plan]


def test_fixture_shape():
    """CPU: the fixtures exist, are 1e6 (or the 1e5 reference legs) and the
    restatement agreed with the reference where it was cross-checked."""
    for name in ("bench", "ns12", "predict"):
        c = FIX[name]
        assert c["trials"] == 1_000_000 and len(c["plan"]) == len(c["n_seq"]) - 1
    assert FIX["bench"]["n_seq"][0] == 256 and len(FIX["bench"]["n_seq"]) == 25
    assert len(FIX["config3"]["replans"]) == 60 and FIX["config3"]["trials"] == 1_000_000
    for name in ("ref_1e5_gpt3_128", "ref_1e5_ns12"):
        assert FIX[name]["trials"] == 100_000 and FIX[name]["reference_plan_equal"] is True


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["bench", "ns12", "predict", "ref_1e5_ns12", "ref_1e5_gpt3_128"])
def test_replan_matches_fixture(name):
    from paper_2403_14097_b200.planner import Planner
    c = FIX[name]
    w = PROFILES[c["profile"]]()
    with Planner(w, CostTable(), PlannerOptions(mc_trials=c["trials"])) as p:
        got = _rows(p.dp_optimize(_cfg(c["current"]), c["n_seq"]))
        assert got == c["plan"], name
        # the prepared (device-resident) path gives the same plan
        p.prepare(_cfg(c["current"]), c["n_seq"])
        p.execute()
        assert _rows(p.fetch(len(c["n_seq"]) - 1)) == c["plan"], name


@pytest.mark.gpu
def test_config3_proactive_replans_with_cache():
    """Config 3 (GPT-3 6.7B, N=128, 1e6): the first 60 Proactive(12, arima)
    re-plans of the replay, one persistent planner with the device histogram
    cache on (the reference's hist_cache_), each re-plan bit-identical."""
    from paper_2403_14097_b200.planner import Planner
    c = FIX["config3"]
    w = PROFILES[c["profile"]]()
    with Planner(w, CostTable(), PlannerOptions(mc_trials=c["trials"])) as p:
        p.set_hist_cache(True)
        for i, r in enumerate(c["replans"]):
            assert _rows(p.dp_optimize(_cfg(r["current"]), r["n_seq"])) == r["plan"], i


@pytest.mark.gpu
def test_materialised_phi_matches_fixtures():
    """The materialised-phi DP path (phi launches per pipeline stage + max-plus
    levels; by default on one GPU when the sampling is short against the DP) on the
    full 1e6 ensembles: forced with LIVEPUT_PHI=1, read once per
    process, so it runs in a subprocess."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    names = ["bench", "ns12", "predict"]
    script = (
        "import json, sys\n"
        f"sys.path.insert(0, {str(root)!r}); sys.path.insert(0, {str(root / 'tests')!r})\n"
        "from conftest import load_golden\n"
        "from paper_2403_14097_b200.model import CostTable, ParallelConfig, PlannerOptions, PROFILES\n"
        "from paper_2403_14097_b200.planner import Planner\n"
        "F = load_golden('plans_1e6'); out = {}\n"
        f"for name in {names!r}:\n"
        "    c = F[name]; cur = None if c['current'] is None else ParallelConfig(*c['current'])\n"
        "    with Planner(PROFILES[c['profile']](), CostTable(), PlannerOptions(mc_trials=c['trials'])) as p:\n"
        "        out[name] = [[None if s.config is None else [s.config.pipelines, s.config.stages],\n"
        "                      s.expected_committed.hex(), s.expected_mig_cost_s.hex()]\n"
        "                     for s in p.dp_optimize(cur, c['n_seq'])]\n"
        "print(json.dumps(out))\n")
    env = dict(os.environ, LIVEPUT_PHI="1")
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    for name in names:
        assert got[name] == FIX[name]["plan"], name
