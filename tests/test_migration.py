"""Migration planning for a realised scenario through the C ABI.

Host code (lp_migration.cpp), so these run without a GPU.  The known answers
restate the reference's own test_migration.cpp cases; the differential tests
compare every field of every move with the reference compiled into
oracle/_ref (skipped where /root/reference and the prebuilt copy are absent).
"""
import random

import pytest

from oracle import oracle as O
from paper_2403_14097_b200.model import CostTable, ParallelConfig, WorkloadProfile, lm_1p5b
from paper_2403_14097_b200.planner import (RollbackRequired, plan_migration, resume_cost,
                                           transition_outcome)

W = lm_1p5b()
COSTS = CostTable()


def vec(n, dead=()):
    v = [0] * n
    for k in dead:
        v[k] = 1
    return v


# ---- known answers (reference tests/test_migration.cpp) ------------------------
def test_no_preemption_same_target_is_free():  # test_migration.cpp:8-18
    plan = plan_migration(ParallelConfig(3, 4), 0, vec(12), ParallelConfig(3, 4), W, COSTS)
    assert plan.kind == "none" and plan.moves == [] and plan.est_cost_s == 0.0
    assert plan.cost(W, COSTS, 0) == 0.0


def test_two_losses_one_reroute():  # :20-32
    v = vec(12, [0 * 4 + 0, 1 * 4 + 1])
    plan = plan_migration(ParallelConfig(3, 4), 0, v, ParallelConfig(2, 4), W, COSTS)
    assert plan.kind == "intra_stage"
    assert len(plan.moves) == 1 and not plan.moves[0].transfers_params
    assert all(not v[m.instance] for m in plan.moves)


def test_fully_preempted_stage_rolls_back():  # :34-42
    v = vec(6, [0 * 3 + 1, 1 * 3 + 1])
    with pytest.raises(RollbackRequired):
        plan_migration(ParallelConfig(2, 3), 0, v, ParallelConfig(1, 3), W, COSTS)


def test_inter_stage_alpha_beta():  # :44-62
    w = lm_1p5b()
    w.param_bytes, w.alpha_s, w.beta_s_per_byte = 3.0e9, 1e-3, 1.0 / 10e9
    v = vec(17, [0 * 8 + 3])  # one hole at stage 3, one spare
    plan = plan_migration(ParallelConfig(2, 8), 1, v, ParallelConfig(2, 8), w, COSTS)
    assert plan.kind == "inter_stage" and plan.transfer_rounds == 1
    transfer = (3.0e9 / 8) * (1.0 / 10e9) + 1e-3
    assert plan.cost(w, COSTS, 0) == pytest.approx(COSTS.build_model_s + COSTS.update_comm_groups_s + transfer)
    assert plan.moves[-1].from_pipeline == -1 and plan.moves[-1].transfers_params  # the spare


def test_pipeline_dominates():  # :64-75
    v = vec(32, [3])
    same = plan_migration(ParallelConfig(4, 8), 0, v, ParallelConfig(3, 8), W, COSTS)
    pipe = plan_migration(ParallelConfig(4, 8), 0, v, ParallelConfig(3, 7), W, COSTS)
    assert pipe.kind == "pipeline" and pipe.est_cost_s > same.est_cost_s


def test_size_mismatch_and_too_few_bodies():
    with pytest.raises(ValueError):
        plan_migration(ParallelConfig(2, 3), 0, vec(5), ParallelConfig(2, 3), W, COSTS)
    with pytest.raises(ValueError):  # one dead slot, no spare, no surplus: the hole cannot be filled
        plan_migration(ParallelConfig(2, 3), 0, vec(6, [1]), ParallelConfig(2, 3), W, COSTS)


def test_costs_ordering_and_transition_outcome_agree():  # :77-110, :139-156
    rng = random.Random(909)
    for _ in range(300):
        d, p, spares = rng.randint(1, 4), rng.randint(2, 5), rng.randint(0, 2)
        n = d * p + spares
        v = [1 if rng.random() < 0.2 else 0 for _ in range(n)]
        surv = [sum(1 for r in range(d) if not v[r * p + s]) for s in range(p)]
        alive = n - sum(v)
        td = min(min(surv), alive // p)
        if td < 1:
            continue
        plan = plan_migration(ParallelConfig(d, p), spares, v, ParallelConfig(td, p), W, COSTS)
        cost, kind, rb = transition_outcome(min(surv + [d]), ParallelConfig(d, p), ParallelConfig(td, p), 0, W,
                                            COSTS)
        assert not rb and plan.kind == kind
        assert plan.cost(W, COSTS, 0) == pytest.approx(cost)
        assert all(not v[m.instance] for m in plan.moves)
    assert resume_cost(ParallelConfig(2, 8), W, COSTS) > 0.0


# ---- differential: every move against the compiled reference -------------------
def _random_profile(rng):
    return WorkloadProfile("rand", rng.uniform(0.1, 2.0), rng.uniform(1e7, 5e9), rng.uniform(0, 1e8), 64, 1,
                           1.0, 0.0, 0.0, rng.uniform(0, 1e-2), rng.uniform(1e-11, 1e-8))


@pytest.mark.skipif(not O.ref_available(), reason="reference library not available")
def test_plan_migration_matches_reference():
    rng = random.Random(20240318)
    kinds = {"none": 0, "intra_stage": 1, "inter_stage": 2, "pipeline": 3}
    seen = set()
    for trial in range(3000):
        w = _random_profile(rng) if trial % 3 else W
        costs = CostTable(*[rng.uniform(0.0, 10.0) for _ in range(6)]) if trial % 5 == 0 else COSTS
        d, p, spares = rng.randint(1, 6), rng.randint(1, 6), rng.randint(0, 4)
        n = d * p + spares
        rate = rng.choice([0.0, 0.1, 0.25, 0.5])
        v = [1 if rng.random() < rate else 0 for _ in range(n)]
        td = rng.randint(0, d + 2)
        tp = p if rng.random() < 0.8 else rng.randint(1, 7)
        src, tgt = ParallelConfig(d, p), ParallelConfig(td, tp)
        ref = O.ref_plan_migration(w, costs, src, spares, v, tgt)
        try:
            got = plan_migration(src, spares, v, tgt, w, costs)
        except RollbackRequired:
            assert ref == ("rollback",), (src, spares, v, tgt, ref)
            seen.add("rollback")
            continue
        except ValueError:
            assert ref == ("invalid",), (src, spares, v, tgt, ref)
            seen.add("invalid")
            continue
        assert ref[0] == "ok", (src, spares, v, tgt, ref)
        _, kind, rounds, moves, est, cost_fresh = ref
        assert kinds[got.kind] == kind and got.transfer_rounds == rounds
        assert [(m.instance, m.from_pipeline, m.from_stage, m.to_pipeline, m.to_stage, int(m.transfers_params))
                for m in got.moves] == moves
        assert got.est_cost_s == est and got.cost(w, costs, 1) == cost_fresh
        seen.add(got.kind)
    assert seen >= {"none", "intra_stage", "inter_stage", "pipeline", "rollback", "invalid"}


@pytest.mark.skipif(not O.ref_available(), reason="reference library not available")
def test_transition_outcome_matches_reference():
    rng = random.Random(7)
    for _ in range(2000):
        w = _random_profile(rng)
        costs = CostTable(*[rng.uniform(0.0, 10.0) for _ in range(6)])
        sd, sp = rng.randint(1, 40), rng.randint(1, 40)
        td, tp = rng.randint(1, 40), sp if rng.random() < 0.7 else rng.randint(1, 40)
        m = rng.randint(0, sd)
        fresh = rng.randint(0, 1)
        cost, kind, rb = transition_outcome(m, ParallelConfig(sd, sp), ParallelConfig(td, tp), fresh, w, costs)
        ref = O.ref_transition_outcome(w, costs, m, sd, sp, td, tp, fresh)
        assert (cost, kind, rb) == ref
