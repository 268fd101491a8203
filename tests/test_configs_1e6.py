"""BASELINE configs 2, 3 and 5 pinned at the sample count they are timed at
(1e6 per point), against tests/golden/configs_1e6.json (the oracle's
strategy sequences; make_configs_1e6.py).  Every re-plan's first step — the
configuration and both FP64 step values — must match bit for bit, through a
persistent planner with the device histogram cache on (the simulator's
shared Planner and the reference's hist_cache_), and the whole simulator run
(lp_simulate at 1e6) must execute exactly those configurations."""
import pytest

from conftest import load_golden
from paper_2403_14097_b200.model import CostTable, ParallelConfig, PlannerOptions, PROFILES

FIX = load_golden("configs_1e6")


def _cfg(x):
    return None if x is None else ParallelConfig(*x)


def _step(s):
    return [None if s.config is None else [s.config.pipelines, s.config.stages], s.expected_committed.hex(),
            s.expected_mig_cost_s.hex()]


def test_fixture_shape():
    assert FIX["config3i"]["trials"] == FIX["config3p"]["trials"] == FIX["config2"]["trials"] == 1_000_000
    assert len(FIX["config3i"]["replans"]) == len(FIX["config3p"]["replans"]) == 1440
    assert len(FIX["config2"]["traces"]) == 5
    assert all(len(v) == 60 for v in FIX["config2"]["traces"].values())


def _replay(profile, replans):
    from paper_2403_14097_b200.planner import Planner
    w = PROFILES[profile]()
    with Planner(w, CostTable(), PlannerOptions(mc_trials=1_000_000)) as p:
        p.set_hist_cache(True)
        for i, r in enumerate(replans):
            plan = p.dp_optimize(_cfg(r["current"]), r["n_seq"])
            assert _step(plan[0]) == r["first"], i


def _sim_configs(profile, counts, pol_name, seed):
    from paper_2403_14097_b200.planner import policy, simulate
    rep, ivs = simulate(counts, PROFILES[profile](), policy(pol_name), seed, PlannerOptions(mc_trials=1_000_000),
                        CostTable(), 60.0, 128 if profile == "lm_6p7b" else 64)
    return [None if iv["pipelines"] == 0 else [iv["pipelines"], iv["stages"]] for iv in ivs]


@pytest.mark.gpu
@pytest.mark.parametrize("name,pol", [("config3i", "ideal"), ("config3p", "proactive")])
def test_config3_replay_1e6(name, pol):
    import json
    from pathlib import Path
    c = FIX[name]
    _replay(c["profile"], c["replans"])
    counts = json.loads((Path(__file__).resolve().parents[1] / c["trace"]).read_text())["counts"]
    assert _sim_configs(c["profile"], counts, pol, 1) == [r["current"] for r in c["replans"]]


@pytest.mark.gpu
def test_config3_gpu_forecasts_equal_fixture_nseq():
    """The Proactive n_seq came from the reference's predict(); the device's
    batched forecasts (lp_predict_windows) reproduce every one of them."""
    import json
    from pathlib import Path
    from paper_2403_14097_b200.planner import ForecastConfig, predict_windows
    c = FIX["config3p"]
    counts = json.loads((Path(__file__).resolve().parents[1] / c["trace"]).read_text())["counts"]
    H = I = 12
    series = [counts[0]] * (H - 1) + counts + [0] * I
    preds, _ = predict_windows(series, ForecastConfig(history_len=H, lookahead=I, capacity=128), ["arima"])
    for i, r in enumerate(c["replans"]):
        assert preds[i][0] == r["n_seq"][1:], i


@pytest.mark.gpu
def test_config2_replay_1e6():
    import json
    from pathlib import Path
    c = FIX["config2"]
    data = json.loads((Path(__file__).resolve().parents[1] / "tools" / "data" /
                       "trace_config2_resnet64.json").read_text())
    for s, replans in c["traces"].items():
        _replay(c["profile"], replans)
        assert _sim_configs(c["profile"], data["traces"][s], "ideal", int(s)) == [r["current"] for r in replans], s


@pytest.mark.gpu
def test_sweep_points_1e6():
    from paper_2403_14097_b200.planner import Planner
    c = FIX["sweep"]
    w = PROFILES[c["profile"]]()
    with Planner(w, CostTable(), PlannerOptions(mc_trials=c["trials"])) as p:
        for pt in c["points"]:
            assert [_step(s) for s in p.dp_optimize(_cfg(pt["current"]), pt["n_seq"])] == pt["plan"], (pt["n"], pt["I"])
