"""CPU: pin the oracle (oracle/liveput_oracle.c) against the reference's golden
vectors (tests/golden, generated from the compiled reference) and, when the
reference library is available, against the reference live."""
import ctypes as C

import numpy as np
import pytest

from conftest import load_golden, profile_by_name, profile_from_dict, unhex
from oracle import oracle as O
from paper_2403_14097_b200.model import CostTable, ParallelConfig, PlannerOptions, lm_1p5b

KNOWN_NSEQ = [32, 28, 28, 26, 29, 26, 26, 21, 23, 23, 21, 25, 22]


def cfg(x):
    return None if x is None else ParallelConfig(*x)


# ---- SURVEY.md §8c known answers ------------------------------------------
def test_known_answer_rng():
    L = O.oracle_lib()
    st = C.c_uint64(0)
    got = [L.or_splitmix_next(C.byref(st)) for _ in range(3)]
    assert got == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    seed_nk = O.planner_seed(0x5EED, 32, 3)
    assert seed_nk == 0xC12CFB4BF0CA8483
    assert O.mix_seed(seed_nk, 0) == 0x5C19EED1F87C78E7
    out = (C.c_int * 3)()
    L.or_sample_distinct(32, 3, 0x5C19EED1F87C78E7, out)
    assert list(out) == [6, 25, 8]
    sc = O.oracle_scenarios(32, 3, False, 4, seed_nk)
    assert sc.tolist() == [[6, 8, 25], [18, 29, 31], [0, 6, 16], [5, 18, 29]]


def test_known_answer_hist_phi_plan():
    w = lm_1p5b()
    op = O.OraclePlanner(w, CostTable(), PlannerOptions(mc_trials=10000))
    counts, tot = op.survivor_counts(ParallelConfig(4, 7), 32, 3)
    assert counts.tolist() == [0, 46, 2412, 7535, 7] and tot == 10000
    assert op.phi(ParallelConfig(4, 7), ParallelConfig(4, 7), 32, 29) == (675.38034536719283, 16.070126642857144)
    assert op.phi(ParallelConfig(4, 7), ParallelConfig(3, 8), 32, 29) == (533.35706340378192, 22.539999999999999)
    assert O.oracle_throughput(w, ParallelConfig(4, 7)) == 15.374056280027453
    assert op.liveput(ParallelConfig(4, 7), 32, 3) == pytest.approx(12.475557718208647, rel=1e-13)
    cur = O.oracle_reactive(w, 32)
    assert cur == ParallelConfig(4, 8)
    plan, value = op.dp_optimize(cur, KNOWN_NSEQ, with_value=True)
    assert [s.config for s in plan] == [ParallelConfig(3, 8)] * 6 + [ParallelConfig(3, 7)] * 6
    assert value == 8460.1874990222786


# ---- golden vectors --------------------------------------------------------
def test_golden_rng():
    g = load_golden("rng")
    L = O.oracle_lib()
    for seed, draws in g["splitmix_draws"].items():
        st = C.c_uint64(int(seed))
        assert [L.or_splitmix_next(C.byref(st)) for _ in range(len(draws))] == draws
    for a, b, v in g["mix_seed"]:
        assert O.mix_seed(a, b) == v
    for c in g["sample_distinct"]:
        out = (C.c_int * max(c["k"], 1))()
        L.or_sample_distinct(c["n"], c["k"], c["seed"], out)
        assert list(out[: c["k"]]) == c["out"]


def test_golden_scenarios():
    g = load_golden("scenarios")
    for c in g["sample_vectors"]:
        sc = O.oracle_scenarios(c["n"], c["k"], False, c["trials"], c["seed"])
        assert sc.tolist() == c["sets"]
    for c in g["enumerate_vectors"]:
        cnt = O.oracle_lib().or_scenario_count(c["n"], c["k"])
        sc = O.oracle_scenarios(c["n"], c["k"], True, cnt, 0)
        assert sc.tolist() == c["sets"]
    for n, k, v in g["scenario_count"]:
        assert O.oracle_lib().or_scenario_count(n, k) == v


def test_golden_survivors():
    for c in load_golden("survivors"):
        cfgs = [ParallelConfig(*x) for x in c["configs"]]
        sc = O.oracle_scenarios(c["n"], c["k"], False, c["trials"], c["seed"])
        m = np.array(c["m"])
        # the oracle's ensemble histogram equals the bincount of the reference's minima
        counts, tot = O.oracle_ensemble_counts(c["n"], c["k"], False, c["trials"], c["seed"], cfgs)
        assert tot == c["trials"]
        for ci, cf in enumerate(cfgs):
            ref = np.bincount(m[:, ci], minlength=counts.shape[1])
            assert counts[ci].tolist() == ref.tolist()
        assert sc.shape == (c["trials"], c["k"])


def test_golden_histograms():
    for c in load_golden("histograms"):
        w = profile_by_name(c["profile"])
        op = O.OraclePlanner(w, CostTable(), PlannerOptions(mc_trials=c["mc_trials"]))
        counts, tot = op.survivor_counts(ParallelConfig(*c["cfg"]), c["n"], c["k"])
        hist = [float(x) / float(tot) for x in counts]
        assert [float.hex(h) for h in hist] == c["hist"], c


def test_golden_phi():
    for c in load_golden("phi"):
        w = profile_by_name(c["profile"])
        op = O.OraclePlanner(w, CostTable(), PlannerOptions(mc_trials=c["mc_trials"], strict_conditional=c["strict"]))
        got = op.phi(cfg(c["prev"]), cfg(c["next"]), c["n_now"], c["n_next"])
        assert got == (unhex(c["committed"]), unhex(c["mig"])), c


def test_golden_plans():
    for c in load_golden("plans"):
        w = profile_by_name(c["profile"])
        op = O.OraclePlanner(w, CostTable(), PlannerOptions(mc_trials=c["mc_trials"], exact_cap=c["exact_cap"],
                                                            strict_conditional=c["strict"]))
        plan = op.dp_optimize(cfg(c["current"]), c["n_seq"])
        got = [[s.interval_index, None if s.config is None else [s.config.pipelines, s.config.stages],
                float.hex(s.expected_committed), float.hex(s.expected_mig_cost_s)] for s in plan]
        assert got == c["plan"], c["tag"]
        seq = [s.config for s in plan]
        assert float.hex(op.sequence_value(cfg(c["current"]), seq, c["n_seq"])) == c["value"]


def test_golden_random_dp():
    for c in load_golden("random_dp"):
        w = profile_from_dict(c["profile"])
        op = O.OraclePlanner(w, CostTable(**c["costs"]), PlannerOptions(**c["options"]))
        plan = op.dp_optimize(cfg(c["current"]), c["n_seq"])
        got = [[s.interval_index, None if s.config is None else [s.config.pipelines, s.config.stages],
                float.hex(s.expected_committed), float.hex(s.expected_mig_cost_s)] for s in plan]
        assert got == c["plan"]


def test_golden_tables():
    g = load_golden("tables")
    for c in g["throughput"]:
        w = profile_by_name(c["profile"])
        assert float.hex(O.oracle_throughput(w, ParallelConfig(*c["cfg"]))) == c["value"]
    for c in g["configs"]:
        w = profile_by_name(c["profile"])
        assert [[x.pipelines, x.stages] for x in O.oracle_configs(w, c["n"])] == c["configs"]
    for c in g["reactive"]:
        r = O.oracle_reactive(profile_by_name(c["profile"]), c["n"])
        assert (None if r is None else [r.pipelines, r.stages]) == c["cfg"]
    L = O.oracle_lib()
    w = lm_1p5b()
    p, keep = w.to_c()
    costs = CostTable().to_c()
    for c in g["transition"]:
        rb, kind = C.c_int(), C.c_int()
        cost = L.or_transition_cost(*c["args"], C.byref(p), C.byref(costs), C.byref(rb), C.byref(kind))
        assert (float.hex(cost), rb.value, kind.value) == (c["cost"], c["rollback"], c["kind"])


# ---- live differential against the compiled reference ----------------------
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference not built/present")


@needs_ref
def test_live_random_phi_and_hist():
    rng = np.random.default_rng(7)
    w = lm_1p5b()
    for trial in range(30):
        n = int(rng.integers(7, 120))
        n2 = int(rng.integers(0, n + 10))
        k = max(0, n - n2)
        opt = PlannerOptions(mc_trials=int(rng.integers(1, 400)), exact_cap=int(rng.choice([0, 50, 2000])))
        rp, op = O.RefPlanner(w, CostTable(), opt), O.OraclePlanner(w, CostTable(), opt)
        cs = O.oracle_configs(w, n)
        ns = O.oracle_configs(w, n2) + [None]
        for _ in range(5):
            a = cs[int(rng.integers(0, len(cs)))]
            b = ns[int(rng.integers(0, len(ns)))]
            assert rp.phi(a, b, n, n2) == op.phi(a, b, n, n2)
            h = rp.survivor_hist(a, n, k)
            cnt, tot = op.survivor_counts(a, n, k)
            assert [float.hex(x) for x in h] == [float.hex(float(x) / tot) for x in cnt]


@needs_ref
def test_live_dp_n96():
    w = lm_1p5b()
    opt = PlannerOptions(mc_trials=300)
    ns = [96, 90, 93, 84, 84, 88, 80, 75]
    cur = O.oracle_reactive(w, 96)
    a = O.RefPlanner(w, CostTable(), opt).dp_optimize(cur, ns)
    b = O.OraclePlanner(w, CostTable(), opt).dp_optimize(cur, ns)
    assert a == b


def test_oracle_memo_identical():
    """The restatement's opt-in per-(n, k) memo (used to generate the long 1e6
    replay fixtures) gives the same plans and values as the cache-free path."""
    import json
    from pathlib import Path
    from oracle.oracle import OraclePlanner
    from paper_2403_14097_b200.model import CostTable, ParallelConfig, PlannerOptions, lm_6p7b
    counts = json.loads((Path(__file__).resolve().parents[1] / "tools" / "data" /
                         "trace_gen_synthetic_128.json").read_text())["counts"]
    w = lm_6p7b()
    opt = PlannerOptions(mc_trials=3000)
    a = OraclePlanner(w, CostTable(), opt, cache=True)
    b = OraclePlanner(w, CostTable(), opt)
    cur = ParallelConfig(3, 20)  # fits every count of the first 60 intervals (>= 66)
    for i in range(0, 60, 6):
        ns = counts[i:i + 13]
        assert a.dp_optimize(cur, ns) == b.dp_optimize(cur, ns), i
