"""The replay driver: lp_simulate restates the reference
simulator's run() around this library's planner and forecasts.  Every field
of the report and of every interval log is compared with the reference's
run() compiled into oracle/_ref (FP64 equality).  The reactive, checkpoint
and redundancy policies never plan, so they run without a GPU; proactive and
ideal plan every interval on the device."""
import pytest

from oracle import oracle as O
from paper_2403_14097_b200.model import CostTable, PlannerOptions, lm_1p5b, lm_6p7b
from paper_2403_14097_b200.planner import policy, simulate, simulate_batch

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not available")


def _traces():
    return [(32, O.ref_gen_synthetic(1, 32, 90, 9, 8, 1, 4)),
            (64, O.ref_gen_synthetic(4, 64, 120, 30, 25, 1, 8)),
            (128, O.ref_gen_synthetic(2, 128, 80, 60, 50, 1, 8))]


def _check(w, name, cap, tr, seed, opt, costs, **kw):
    pol = policy(name, **kw)
    got = simulate(tr, w, pol, seed, opt, costs, interval_s=60.0, capacity=cap, spot_price_per_hour=0.9,
                   ondemand_price_per_hour=3.1)
    ref = O.ref_simulate(tr, w, pol, seed, opt, costs, 60.0, cap, 0, 0.9, 3.1)
    assert got[0] == ref[0], (name, cap, seed)
    assert got[1] == ref[1], (name, cap, seed)
    return got


@needs_ref
def test_non_planning_policies_match_reference():
    opt = PlannerOptions(mc_trials=1000)
    for w in (lm_1p5b(), lm_6p7b()):
        for cap, tr in _traces():
            for seed in (1, 7):
                for name, kw in [("reactive", {}), ("checkpoint", {}), ("checkpoint", {"ckpt_period_intervals": 3}),
                                 ("redundancy", {"redundancy_fixed_stages": 8}), ("redundancy", {})]:
                    rep, _ = _check(w, name, cap, tr, seed, opt, CostTable(), **kw)
                    assert rep["sample_accounting_ok"]


@needs_ref
@pytest.mark.gpu
def test_planning_policies_match_reference():
    opt = PlannerOptions(mc_trials=1000)
    w = lm_1p5b()
    for cap, tr in _traces():
        for name in ("ideal", "proactive"):
            rep, ivs = _check(w, name, cap, tr, 3, opt, CostTable())
            assert len(ivs) == len(tr)
    rep, _ = _check(lm_6p7b(), "proactive", 128, _traces()[2][1], 5, opt, CostTable(), method="moving_avg")


@pytest.mark.gpu
def test_batch_equals_single_runs():
    """One planning pass for many seeds gives each seed's own run()."""
    opt = PlannerOptions(mc_trials=2000)
    cap, tr = _traces()[1]
    for name in ("proactive", "checkpoint"):
        pol = policy(name)
        seeds = [1, 2, 3, 99]
        batch = simulate_batch(tr, lm_1p5b(), pol, seeds, opt, CostTable(), capacity=cap)
        for s, got in zip(seeds, batch):
            assert got == simulate(tr, lm_1p5b(), pol, s, opt, CostTable(), capacity=cap)


def test_batch_non_planning_equals_single_runs():
    """The batch entry point for the policies that never plan (CPU only)."""
    opt = PlannerOptions(mc_trials=1000)
    cap, tr = 64, [64, 60, 61, 55, 58, 50, 50, 47, 52, 49, 40, 44, 48, 48, 45, 30, 35, 44, 50, 52]
    for name in ("reactive", "checkpoint"):
        pol = policy(name)
        seeds = [3, 4, 5]
        batch = simulate_batch(tr, lm_1p5b(), pol, seeds, opt, CostTable(), capacity=cap)
        for s, got in zip(seeds, batch):
            assert got == simulate(tr, lm_1p5b(), pol, s, opt, CostTable(), capacity=cap)
            assert got[0]["seed"] == s
