"""GPU parity: libliveput.so (sm_100a) against the reference's golden vectors and
the CPU oracle, through the C ABI.  Integer results (scenarios, survivor
minima, histogram counts) and the strategy sequence must match bit-exactly;
FP64 phi / plan values are bit-exact too (tolerance 0) because every device
FP64 op is an explicit round-to-nearest intrinsic in the reference's order.
expected_liveput sums in a different order: tolerance 1e-12 relative."""
import numpy as np
import pytest

from conftest import load_golden, profile_by_name, profile_from_dict, unhex
from oracle import oracle as O
from paper_2403_14097_b200.model import (CostTable, ParallelConfig, PlannerOptions, lm_1p5b, lm_6p7b,
                                         resnet152_dp, toy_six_instance)

pytestmark = pytest.mark.gpu

KNOWN_NSEQ = [32, 28, 28, 26, 29, 26, 26, 21, 23, 23, 21, 25, 22]


def cfg(x):
    return None if x is None else ParallelConfig(*x)


def planner(w, opt=None, costs=None):
    from paper_2403_14097_b200.planner import Planner
    return Planner(w, costs or CostTable(), opt or PlannerOptions())


def plan_rows(plan):
    return [[s.interval_index, None if s.config is None else [s.config.pipelines, s.config.stages],
             float.hex(s.expected_committed), float.hex(s.expected_mig_cost_s)] for s in plan]


@pytest.fixture(scope="module")
def gpt2():
    p = planner(lm_1p5b(), PlannerOptions(mc_trials=10000))
    yield p
    p.close()


def test_native_library_is_in_tree():
    from paper_2403_14097_b200 import _abi
    lib = _abi.lib()
    assert str(_abi.LIB_PATH).endswith("paper_2403_14097_b200/lib/libliveput.so")
    assert "sm_100a" in lib.lp_build_info().decode()


# ---- scenario generation ---------------------------------------------------
def test_scenarios_match_reference_sample_vectors(gpt2):
    for c in load_golden("scenarios")["sample_vectors"]:
        got = gpt2.dump_scenarios(c["n"], c["k"], c["trials"], c["seed"])
        assert got.astype(int).tolist() == c["sets"], (c["n"], c["k"])


def test_known_answer_trials(gpt2):
    seed = O.planner_seed(0x5EED, 32, 3)
    got = gpt2.dump_scenarios(32, 3, 4, seed)
    assert got.tolist() == [[6, 8, 25], [18, 29, 31], [0, 6, 16], [5, 18, 29]]


def test_survivor_minima_match_reference(gpt2):
    for c in load_golden("survivors"):
        cfgs = [ParallelConfig(*x) for x in c["configs"]]
        got = gpt2.dump_survivors(c["n"], c["k"], c["trials"], c["seed"], cfgs)
        assert got.astype(int).tolist() == c["m"], (c["profile"], c["n"], c["k"])


def test_exact_enumeration_order(gpt2):
    for c in load_golden("scenarios")["enumerate_vectors"]:
        if c["k"] == 0:
            continue
        cnt = len(c["sets"])
        cfgs = [ParallelConfig(1, 1)]
        got = gpt2.dump_survivors(c["n"], c["k"], cnt, 0, cfgs, exact=True)
        # survivors of config (1,1): 0 iff slot 0 preempted
        assert got[:, 0].tolist() == [0 if s[0] == 0 else 1 for s in c["sets"]]


# ---- histograms ----------------------------------------------------------------
def test_histograms_match_reference():
    by = {}
    for c in load_golden("histograms"):
        by.setdefault((c["profile"], c["mc_trials"]), []).append(c)
    for (prof, trials), cases in by.items():
        p = planner(profile_by_name(prof), PlannerOptions(mc_trials=trials))
        for c in cases:
            h = p.survivor_histogram(ParallelConfig(*c["cfg"]), c["n"], c["k"])
            assert [float.hex(x) for x in h] == c["hist"], c
        p.close()


def test_known_answer_histogram(gpt2):
    counts, tot = gpt2.survivor_counts(ParallelConfig(4, 7), 32, 3)
    assert counts.tolist() == [0, 46, 2412, 7535, 7] and tot == 10000


@pytest.mark.parametrize("seed", range(6))
def test_random_ensembles_vs_oracle(seed):
    """Both kernel variants (k <= 16 registers, k > 16 counters), random n/k,
    every config of n, bit-exact counts."""
    rng = np.random.default_rng(1000 + seed)
    for prof in ("lm_1p5b", "resnet152", "lm_6p7b"):
        w = profile_by_name(prof)
        n = int(rng.integers(20, 520))
        k = int(rng.choice([1, 2, 3, 5, 8, 11, 16, 17, 24, 40, 63, min(n - 1, 100)]))
        k = min(k, n)
        trials = int(rng.integers(500, 5000))
        opt = PlannerOptions(mc_trials=trials, exact_cap=0)
        p = planner(w, opt)
        cs = O.oracle_configs(w, n)
        if not cs:
            p.close()
            continue
        sel = [cs[i] for i in sorted(set(rng.integers(0, len(cs), 12).tolist()))]
        ref, tot = O.oracle_ensemble_counts(n, k, False, trials, O.planner_seed(0x5EED, n, k), sel)
        for ci, c in enumerate(sel):
            got, gt = p.survivor_counts(c, n, k)
            assert gt == tot
            assert got.tolist() == ref[ci][: c.pipelines + 1].tolist(), (prof, n, k, c)
        p.close()


def test_exact_branch_counts_vs_oracle():
    w = lm_1p5b()
    p = planner(w, PlannerOptions(exact_cap=1000000))
    for n, k in [(64, 2), (40, 3), (20, 10), (21, 18), (30, 29), (12, 0), (9, 9), (100, 1)]:
        cs = O.oracle_configs(w, n)
        if not cs:
            continue
        ref, tot = O.oracle_ensemble_counts(n, k, True, 0, 0, cs)
        for ci, c in enumerate(cs):
            got, gt = p.survivor_counts(c, n, k)
            assert gt == tot and got.tolist() == ref[ci][: c.pipelines + 1].tolist(), (n, k, c)
    p.close()


def test_slot_walk_depths_vs_oracle():
    """9 <= k <= 16 at depths P <= 16 with 10..64 rows take the register slot
    walk (lp_hist_rows.cu walk_elems), P = 1 included; MC and exact branches,
    every config, bit-exact counts."""
    w = resnet152_dp()
    cases = [(40, 9, False), (100, 12, False), (300, 16, False), (160, 16, False), (64, 13, False),
             (20, 10, True), (22, 11, True), (30, 12, False)]
    for n, k, exact in cases:
        trials = 3000
        opt = PlannerOptions(mc_trials=trials, exact_cap=1000000 if exact else 0)
        p = planner(w, opt)
        cs = [c for c in O.oracle_configs(w, n) if c.stages <= 20]
        ref, tot = O.oracle_ensemble_counts(n, k, exact, trials, O.planner_seed(0x5EED, n, k), cs)
        for ci, c in enumerate(cs):
            got, gt = p.survivor_counts(c, n, k)
            assert gt == tot and got.tolist() == ref[ci][: c.pipelines + 1].tolist(), (n, k, exact, c)
        p.close()


def test_table_generator_vs_oracle():
    """k > 16 at n <= 256 draws through the byte position table
    (lp_device.cuh gen_mc_bitmap_tab); n > 256 through the displacement list.
    Every config, bit-exact counts, up to k = n - 1."""
    w = resnet152_dp()
    for n, k in [(256, 17), (256, 40), (200, 64), (129, 100), (256, 255), (64, 63), (300, 40), (257, 33)]:
        trials = 2000
        opt = PlannerOptions(mc_trials=trials, exact_cap=0)
        p = planner(w, opt)
        cs = O.oracle_configs(w, n)
        cs = cs[:: max(1, len(cs) // 60)]
        ref, tot = O.oracle_ensemble_counts(n, k, False, trials, O.planner_seed(0x5EED, n, k), cs)
        for ci, c in enumerate(cs):
            got, gt = p.survivor_counts(c, n, k)
            assert gt == tot and got.tolist() == ref[ci][: c.pipelines + 1].tolist(), (n, k, c)
        p.close()


def test_maximum_size_ensembles_vs_oracle():
    """n = kMaxN = 2048 (the scenario-major kernel past n = 512), sparse and
    dense preemption, and a re-plan at n = 1024 against the cache-free oracle."""
    w = resnet152_dp()
    assert O.oracle_configs(w, 2048)
    for n, k in [(2048, 20), (2048, 200), (1500, 5)]:
        trials = 2000
        p = planner(w, PlannerOptions(mc_trials=trials, exact_cap=0))
        cs = O.oracle_configs(w, n)
        sel = cs[:: max(1, len(cs) // 12)]
        ref, tot = O.oracle_ensemble_counts(n, k, False, trials, O.planner_seed(0x5EED, n, k), sel)
        for ci, c in enumerate(sel):
            got, gt = p.survivor_counts(c, n, k)
            assert gt == tot and got.tolist() == ref[ci][: c.pipelines + 1].tolist(), (n, k, c)
        p.close()
    ns = [1024, 1000, 1010]
    opt = PlannerOptions(mc_trials=1000)
    cur = O.oracle_reactive(w, ns[0])
    ref = O.OraclePlanner(w, CostTable(), opt).dp_optimize(cur, ns)
    p = planner(w, opt)
    assert plan_rows(p.dp_optimize(cur, ns)) == plan_rows(ref)
    p.close()


# ---- phi, plans ---------------------------------------------------------------
def test_phi_matches_reference():
    for c in load_golden("phi"):
        p = planner(profile_by_name(c["profile"]),
                    PlannerOptions(mc_trials=c["mc_trials"], strict_conditional=c["strict"]))
        v = p.phi(cfg(c["prev"]), cfg(c["next"]), c["n_now"], c["n_next"])
        assert (v.committed, v.mig_cost_s) == (unhex(c["committed"]), unhex(c["mig"])), c
        p.close()


def test_known_answer_plan(gpt2):
    plan = gpt2.dp_optimize(ParallelConfig(4, 8), KNOWN_NSEQ)
    assert [s.config for s in plan] == [ParallelConfig(3, 8)] * 6 + [ParallelConfig(3, 7)] * 6
    v = gpt2.sequence_value(ParallelConfig(4, 8), [s.config for s in plan], KNOWN_NSEQ)
    assert v == 8460.1874990222786


def test_plans_match_reference():
    for c in load_golden("plans"):
        p = planner(profile_by_name(c["profile"]),
                    PlannerOptions(mc_trials=c["mc_trials"], exact_cap=c["exact_cap"],
                                   strict_conditional=c["strict"]))
        plan = p.dp_optimize(cfg(c["current"]), c["n_seq"])
        assert plan_rows(plan) == c["plan"], c["tag"]
        assert float.hex(p.sequence_value(cfg(c["current"]), [s.config for s in plan], c["n_seq"])) == c["value"]
        p.close()


def test_random_small_dp_match_reference():
    for c in load_golden("random_dp"):
        p = planner(profile_from_dict(c["profile"]), PlannerOptions(**c["options"]), CostTable(**c["costs"]))
        assert plan_rows(p.dp_optimize(cfg(c["current"]), c["n_seq"])) == c["plan"]
        p.close()


@pytest.mark.parametrize("case", range(4))
def test_large_replans_vs_oracle(case):
    """N=256..512 re-plans (MC branch, both kernel variants, multi-work-item
    splits) against the cache-free oracle; beyond N=256 the reference's phi
    cache aliases, so the oracle is the checker there."""
    w = [lm_1p5b(), lm_1p5b(), resnet152_dp(), lm_6p7b()][case]
    n_seq = [[256, 224, 224, 208, 232, 208, 208, 168, 184],
             [512, 480, 488, 470, 470, 500, 430],
             [64, 40, 52, 30, 61, 44, 44, 20],
             [128, 120, 121, 110, 118, 104, 104, 96, 100]][case]
    trials = [2000, 500, 3000, 4000][case]
    opt = PlannerOptions(mc_trials=trials)
    cur = O.oracle_reactive(w, n_seq[0])
    ref = O.OraclePlanner(w, CostTable(), opt).dp_optimize(cur, n_seq)
    p = planner(w, opt)
    got = p.dp_optimize(cur, n_seq)
    assert plan_rows(got) == plan_rows(ref)
    p.close()


def test_liveput_table_and_expected_liveput():
    g = load_golden("tables")["liveput"]
    for c in g:
        p = planner(profile_by_name(c["profile"]))
        v = p.expected_liveput(ParallelConfig(*c["cfg"]), c["n"], c["k"], bool(c["exact"]), c["trials"], c["seed"])
        assert v == pytest.approx(unhex(c["value"]), rel=1e-12, abs=1e-12), c
        p.close()
    w = lm_1p5b()
    opt = PlannerOptions(mc_trials=3000)
    p = planner(w, opt)
    op = O.OraclePlanner(w, CostTable(), opt)
    ns = [64, 60, 60, 57]
    p.dp_optimize(ParallelConfig(8, 8), ns, want_liveput=True)
    rows = p.last_liveput
    assert len(rows) == 1 + len(O.oracle_configs(w, 60)) * 2
    for r in rows[:40]:
        k = max(0, ns[r.interval] - ns[r.interval + 1])
        assert r.liveput == pytest.approx(op.liveput(r.config, ns[r.interval], k), rel=1e-12)
    p.close()


# ---- edge cases and errors ---------------------------------------------------
def test_edge_cases_vs_oracle():
    w = toy_six_instance()
    for opt in (PlannerOptions(exact_cap=0, mc_trials=50), PlannerOptions(exact_cap=100000),
                PlannerOptions(mc_trials=1, exact_cap=1)):
        p = planner(w, opt)
        op = O.OraclePlanner(w, CostTable(), opt)
        for cur, ns in [(ParallelConfig(2, 3), [6, 6, 0, 6]), (ParallelConfig(2, 3), [6, 0, 0]),
                        (None, [0, 0, 6]), (ParallelConfig(3, 2), [6, 6]), (ParallelConfig(1, 2), [6, 1, 2, 6, 6, 5])]:
            assert plan_rows(p.dp_optimize(cur, ns)) == plan_rows(op.dp_optimize(cur, ns)), (opt, cur, ns)
        p.close()


def test_errors():
    from paper_2403_14097_b200._abi import LiveputError
    p = planner(lm_1p5b())
    with pytest.raises(ValueError):
        p.dp_optimize(None, [32])
    with pytest.raises(ValueError):
        p.dp_optimize(ParallelConfig(4, 8), [16, 16])  # current exceeds n_seq[0]
    with pytest.raises(ValueError):
        p.sequence_value(None, [None], [8, 8, 8])
    with pytest.raises(LiveputError):
        p.dp_optimize(None, [20000, 19990])  # n beyond kMaxN = 16384: LP_EUNSUPPORTED
    p.close()
    p = planner(lm_1p5b(), PlannerOptions(mc_trials=0))
    with pytest.raises(ValueError):
        p.dp_optimize(ParallelConfig(4, 8), [32, 28])  # sample_vectors: trials must be >= 1
    p.close()
    p = planner(lm_1p5b(), PlannerOptions(exact_cap=10**12))
    with pytest.raises(ValueError):
        p.dp_optimize(ParallelConfig(4, 8), [64, 59])  # C(64,5) in (1e6, exact_cap]: enumerate_vectors throws
    p.close()


def test_full_size_properties():
    """BASELINE config 4 shape (N=256, I=24, 1e6 samples): integer histograms
    sum to the trial count and the plan is deterministic across runs."""
    from bench import north_star_nseq
    w = lm_1p5b()
    p = planner(w, PlannerOptions(mc_trials=1000000))
    ns = north_star_nseq(256, 24)
    cur = O.oracle_reactive(w, ns[0])
    a = p.dp_optimize(cur, ns)
    st = p.stats()
    assert st.resolutions > 5e9
    b = p.dp_optimize(cur, ns)
    assert plan_rows(a) == plan_rows(b)
    for c in [ParallelConfig(32, 7), ParallelConfig(2, 80), ParallelConfig(1, 224)]:
        counts, tot = p.survivor_counts(c, 224, 16)
        assert int(counts.sum()) == tot == 1000000
    p.close()


# ---- device-resident histogram cache (the reference's hist_cache_) ---------
def test_hist_cache_replay_matches_cold():
    """Planning-loop replay (tools/replay.py, Ideal(12)) with the cache on is
    bit-identical to cold re-plans and to the reference's replay fixture."""
    import json
    from pathlib import Path
    from tools.replay import TRACE, loop
    from paper_2403_14097_b200.planner import reactive_plan
    counts = json.loads(Path(TRACE).read_text())["counts"]
    w = lm_6p7b()
    opt = PlannerOptions(mc_trials=1000)
    warm = planner(w, opt)
    warm.set_hist_cache(True)
    cold = planner(w, opt)
    a, _ = loop(warm.dp_optimize, lambda n: reactive_plan(n, w), counts, 300)
    b, _ = loop(cold.dp_optimize, lambda n: reactive_plan(n, w), counts, 300)
    assert a == b
    ref = json.loads((Path(TRACE).parents[2] / "profiles" / "replay_ref_1e3.json").read_text())["sequence"]
    assert a == ref[:300]
    assert warm.stats().cached_pairs >= 0
    warm.close()
    cold.close()


def test_hist_cache_reuses_ensembles():
    w = lm_1p5b()
    p = planner(w, PlannerOptions(mc_trials=20000))
    p.set_hist_cache(True)
    ns = [64, 60, 60, 57, 62, 56]
    a = p.dp_optimize(ParallelConfig(8, 8), ns)
    first = p.stats()
    b = p.dp_optimize(ParallelConfig(8, 8), ns)
    second = p.stats()
    assert plan_rows(a) == plan_rows(b)
    assert first.cached_pairs == 0 and first.mc_pairs > 0
    assert second.mc_pairs == 0 and second.cached_pairs > 0  # everything came from the cache
    p.close()


def test_offline_tables_roundtrip():
    """precompute (n, k) tables, export, import into a fresh
    handle: the re-plan is DP-only and identical to a cold one."""
    w = lm_1p5b()
    opt = PlannerOptions(mc_trials=5000)
    ns = [96, 90, 90, 84, 88, 80]
    pairs = sorted({(ns[j], max(0, ns[j] - ns[j + 1])) for j in range(len(ns) - 1)})
    a = planner(w, opt)
    a.precompute(pairs)
    blob = a.export_tables()
    assert blob[:4] == b"LPC1" and len(blob) > 1000
    b = planner(w, opt)
    b.import_tables(blob)
    cur = ParallelConfig(12, 8)
    warm = b.dp_optimize(cur, ns)
    st = b.stats()
    cold = planner(w, opt).dp_optimize(cur, ns)
    assert plan_rows(warm) == plan_rows(cold)
    assert st.cached_pairs >= 1 and st.mc_pairs <= 1  # only level 0 (current) may need sampling
    c = planner(w, PlannerOptions(mc_trials=5001))
    with pytest.raises(ValueError):
        c.import_tables(blob)
    for p in (a, b, c):
        p.close()


def _decode_tables(blob):
    """lp_cache_export layout (lp_api.cpp CacheHeader / SlotHeader / EntryHeader):
    yields (n, k, count, P, Dmax, probabilities by D: list of min(k,D)+1 by deficit)."""
    import struct
    magic, trials, cap, seed, slots = struct.unpack_from("<IiQQQ", blob, 0)
    assert magic == 0x3143504C
    o = 32
    for _ in range(slots):
        n, k, count, ents, _pad = struct.unpack_from("<iiQii", blob, o)
        o += 24
        for _ in range(ents):
            P, dmax, ln = struct.unpack_from("<iiq", blob, o)
            o += 16
            vals = struct.unpack_from(f"<{ln}d", blob, o)
            o += 8 * ln
            rows, i = [], 0
            for D in range(1, dmax + 1):
                w = min(k, D) + 1
                rows.append(vals[i:i + w])
                i += w
            assert i == ln
            yield n, k, count, P, dmax, rows
    assert o == len(blob)


def test_offline_tables_match_oracle():
    """SURVEY §8f #2 pinned to the oracle: every exported probability
    p(n, k, D, P, m) equals the oracle's count_m / count bit for bit
    (optimizer.cpp:92 normalisation), and a re-plan served from the imported
    tables equals the oracle's plan."""
    w = lm_1p5b()
    opt = PlannerOptions(mc_trials=7000)
    ns = [80, 74, 74, 70, 73, 66]
    pairs = sorted({(ns[j], max(0, ns[j] - ns[j + 1])) for j in range(len(ns) - 1)})
    a = planner(w, opt)
    a.precompute(pairs)
    blob = a.export_tables()
    seen = set()
    for n, k, count, P, dmax, rows in _decode_tables(blob):
        seen.add((n, k))
        exact = O.oracle_lib().or_scenario_count(n, k) <= opt.exact_cap
        cfgs = [ParallelConfig(D, P) for D in range(1, dmax + 1)]
        counts, tot = O.oracle_ensemble_counts(n, k, exact, opt.mc_trials, O.planner_seed(0x5EED, n, k), cfgs)
        assert tot == count
        for D, row in zip(range(1, dmax + 1), rows):
            want = [float(counts[D - 1][D - d]) / float(tot) for d in range(min(k, D) + 1)]
            assert [x.hex() for x in row] == [x.hex() for x in want], (n, k, D, P)
    assert seen == set(pairs)
    b = planner(w, opt)
    b.import_tables(blob)
    cur = ParallelConfig(10, 8)
    got = plan_rows(b.dp_optimize(cur, ns))
    assert got == plan_rows(O.OraclePlanner(w, CostTable(), opt).dp_optimize(cur, ns))
    a.close()
    b.close()


def test_infeasible_current_depth_keeps_later_levels():
    """a level-0 `current` at a depth below the feasible minimum
    (P=3 < 7 for lm_1p5b) with D=1, whose (n, k) ensemble is also read by a
    later level: every feasible depth must keep its t >= 2 events."""
    w = lm_1p5b()
    opt = PlannerOptions(mc_trials=20000)
    for cur, ns in [(ParallelConfig(1, 3), [64, 56, 64, 56, 64, 56]),
                    (ParallelConfig(2, 5), [96, 84, 90, 96, 84, 80]),
                    (ParallelConfig(1, 1), [48, 40, 48, 40])]:
        p = planner(w, opt)
        got = plan_rows(p.dp_optimize(cur, ns))
        ref = plan_rows(O.OraclePlanner(w, CostTable(), opt).dp_optimize(cur, ns))
        assert got == ref, (cur, ns)
        p.close()


@pytest.mark.parametrize("n,k", [(512, 300), (600, 300), (700, 420)])
def test_k_above_255_matches_oracle(n, k):
    """No k cap: more than 255 of n preempted with more than 255
    pipelines per depth — the row kernel at n <= 512 (up to 10 bit planes),
    the scenario-major kernel above (12-bit class counts)."""
    w = resnet152_dp()  # P = 1 is feasible: depth 1 holds n pipelines
    opt = PlannerOptions(mc_trials=3000)
    p = planner(w, opt)
    seed = O.planner_seed(0x5EED, n, k)
    for c in [ParallelConfig(n, 1), ParallelConfig(n // 2, 2), ParallelConfig(n // 3, 3), ParallelConfig(n // 7, 7)]:
        got, tot = p.survivor_counts(c, n, k)
        want, wt = O.oracle_ensemble_counts(n, k, False, opt.mc_trials, seed, [c])
        assert tot == wt and got.tolist() == want[0][: c.pipelines + 1].tolist(), c
    ns = [n, n - k, n - k + 20]
    plan = plan_rows(p.dp_optimize(ParallelConfig(n // 4, 4), ns))
    assert plan == plan_rows(O.OraclePlanner(w, CostTable(), opt).dp_optimize(ParallelConfig(n // 4, 4), ns))
    p.close()


@pytest.mark.parametrize("n,k", [(3000, 5), (3000, 60), (4096, 1500), (16384, 24)])
def test_beyond_2048_instances_vs_oracle(n, k):
    """n up to 16384 (n > 2048 was refused): the global-scratch
    kernel (lp_hist_big.cu) against the cache-free oracle, and a one-interval
    re-plan at n = 3000."""
    w = resnet152_dp()
    trials = 600
    p = planner(w, PlannerOptions(mc_trials=trials, exact_cap=0))
    sel = [ParallelConfig(n, 1), ParallelConfig(n // 2, 2), ParallelConfig(n // 13, 13), ParallelConfig(7, n // 7),
           ParallelConfig(1, n)]
    ref, tot = O.oracle_ensemble_counts(n, k, False, trials, O.planner_seed(0x5EED, n, k), sel)
    for ci, c in enumerate(sel):
        got, gt = p.survivor_counts(c, n, k)
        assert gt == tot and got.tolist() == ref[ci][: c.pipelines + 1].tolist(), (n, k, c)
    p.close()
    if n == 3000:
        opt = PlannerOptions(mc_trials=300)
        ns = [n, n - k]
        cur = ParallelConfig(n // 10, 10)
        want = plan_rows(O.OraclePlanner(w, CostTable(), opt).dp_optimize(cur, ns))
        q = planner(w, opt)
        assert plan_rows(q.dp_optimize(cur, ns)) == want
        q.close()


@pytest.mark.parametrize("n,k", [(1500, 12), (2048, 16), (700, 9)])
def test_large_n_mid_k_vs_oracle(n, k):
    """512 < n <= 2048 with 9 <= k <= 16 runs the bits kernel (round 1 used the
    first-generation dense kernel here): counts of sampled configs against the
    oracle."""
    w = resnet152_dp()
    trials = 3000
    p = planner(w, PlannerOptions(mc_trials=trials, exact_cap=0))
    cs = O.oracle_configs(w, n)
    sel = cs[:: max(1, len(cs) // 16)] + [ParallelConfig(n, 1), ParallelConfig(n // 2, 2)]
    ref, tot = O.oracle_ensemble_counts(n, k, False, trials, O.planner_seed(0x5EED, n, k), sel)
    for ci, c in enumerate(sel):
        got, gt = p.survivor_counts(c, n, k)
        assert gt == tot and got.tolist() == ref[ci][: c.pipelines + 1].tolist(), (n, k, c)
    p.close()
