"""The multi-GPU decomposition through the product path on one GPU.

lp_set_shard makes lp_survivor_hist count one trial slice
[count*r/N, count*(r+1)/N) — the slice rank r of an N-GPU re-plan generates
(lp_api.cpp build_hist_plan t_lo/t_hi, finalize with the local ensemble
size).  Each slice must equal the oracle's counts over the same scenario
ranks bit for bit, and the slices must sum to the single-GPU counts
(integer addition: what ncclAllReduce(sum, u32) computes on N GPUs)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2403_14097_b200.model import CostTable, ParallelConfig, PlannerOptions, lm_1p5b, resnet152_dp

pytestmark = pytest.mark.gpu

CASES = [  # profile, n, k, trials, configs
    (lm_1p5b, 256, 24, 1_000_000, [(32, 8), (2, 80), (1, 224), (36, 7)]),
    (lm_1p5b, 224, 6, 100_003, [(28, 8), (3, 70), (11, 20)]),
    (resnet152_dp, 64, 12, 30_001, [(64, 1), (8, 8), (2, 31), (21, 3)]),
    (lm_1p5b, 40, 3, 1000, [(5, 8), (1, 40)]),  # exact branch: C(40,3) ranks
]


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_shard_slices_match_oracle_and_sum(case, world):
    from paper_2403_14097_b200.planner import Planner
    prof, n, k, trials, cfgs = CASES[case]
    w = prof()
    opt = PlannerOptions(mc_trials=trials)
    exact = O.oracle_lib().or_scenario_count(n, k) <= opt.exact_cap
    count = O.oracle_lib().or_scenario_count(n, k) if exact else trials
    seed = O.planner_seed(0x5EED, n, k)
    with Planner(w, CostTable(), opt) as full, Planner(w, CostTable(), opt) as p:
        for D, P in cfgs:
            c = ParallelConfig(D, P)
            whole, tot = full.survivor_counts(c, n, k)
            acc = np.zeros_like(whole)
            for r in range(world):
                p.set_shard(r, world)
                part, ptot = p.survivor_counts(c, n, k)
                lo, hi = count * r // world, count * (r + 1) // world
                assert ptot == hi - lo
                if trials <= 100_003 or r == 0:  # oracle per slice (1e6 slices: rank 0 only, for time)
                    oc, otot = O.oracle_ensemble_counts_range(n, k, exact, trials if not exact else 0, seed, [c],
                                                              lo, hi)
                    assert otot == ptot and part.tolist() == oc[0][: D + 1].tolist(), (D, P, r)
                acc += part
            assert acc.tolist() == whole.tolist() and tot == count, (D, P)
