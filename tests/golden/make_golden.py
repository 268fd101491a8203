"""Generate tests/golden/*.json from the UNMODIFIED reference (spotsim, compiled
from /root/reference by oracle/Makefile into oracle/_ref/libspotsim_ref.so).

Run in the dev container (the GPU box has no /root/reference):
    python tests/golden/make_golden.py

Floats are stored as float.hex() strings so comparisons are bit-exact.
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from oracle.oracle import RefPlanner, ref_lib  # noqa: E402
from paper_2403_14097_b200.model import (CostTable, ParallelConfig, PlannerOptions,  # noqa: E402
                                         lm_1p5b, lm_6p7b, resnet152_dp, toy_six_instance)

OUT = Path(__file__).resolve().parent
H = float.hex

PROFILES = {"lm_1p5b": lm_1p5b(), "lm_6p7b": lm_6p7b(), "toy_six_instance": toy_six_instance(),
            "resnet152": resnet152_dp()}


def cfgs_of(w, n):
    L = ref_lib()
    p, keep = w.to_c()
    cnt = L.ref_enumerate_configs(C.byref(p), n, None, 0)
    out = (C.c_int * max(2 * cnt, 2))()
    L.ref_enumerate_configs(C.byref(p), n, out, cnt)
    return [ParallelConfig(out[2 * i], out[2 * i + 1]) for i in range(cnt)]


def rng_section():
    L = ref_lib()
    seeds = [0, 1, 0x5EED, 0xDEADBEEF, 2**64 - 1]
    draws = {}
    for s in seeds:
        out = (C.c_uint64 * 8)()
        L.ref_rng_draws(s, 8, out)
        draws[str(s)] = [int(x) for x in out]
    mix = [[a, b, int(L.ref_mix_seed(a, b))] for a, b in
           [(0x5EED, 32), (L.ref_mix_seed(0x5EED, 32), 3), (0, 0), (12345, 2**40), (2**63, 7)]]
    sd = []
    for n, k, seed in [(32, 3, 0x5C19EED1F87C78E7), (8, 8, 1), (100, 17, 7), (256, 40, 99),
                       (512, 1, 3), (5, 0, 9), (2048, 16, 11)]:
        out = (C.c_int * max(k, 1))()
        assert L.ref_sample_distinct(n, k, seed, out) == 0
        sd.append({"n": n, "k": k, "seed": seed, "out": list(out[:k])})
    return {"splitmix_draws": draws, "mix_seed": mix, "sample_distinct": sd}


def scenarios_section():
    L = ref_lib()
    res = []
    for n, k, trials, seed in [(32, 3, 64, None), (8, 3, 50, 42), (64, 9, 40, 5), (256, 8, 32, None),
                               (256, 40, 16, 1234), (100, 17, 16, 77), (6, 6, 4, 3), (2048, 12, 8, 5)]:
        if seed is None:
            seed = int(L.ref_mix_seed(L.ref_mix_seed(0x5EED, n), k))
        buf = (C.c_uint8 * (trials * n))()
        assert L.ref_sample_vectors(n, k, trials, seed, buf) == 0
        v = np.frombuffer(buf, dtype=np.uint8).reshape(trials, n)
        res.append({"n": n, "k": k, "trials": trials, "seed": seed,
                    "sets": [np.nonzero(row)[0].tolist() for row in v]})
    enum = []
    for n, k in [(6, 2), (7, 3), (5, 0), (4, 4), (10, 3)]:
        cnt = int(L.ref_scenario_count(n, k))
        buf = (C.c_uint8 * max(cnt * n, 1))()
        assert L.ref_enumerate_vectors(n, k, buf, cnt) == cnt
        v = np.frombuffer(buf, dtype=np.uint8)[: cnt * n].reshape(cnt, n)
        enum.append({"n": n, "k": k, "sets": [np.nonzero(row)[0].tolist() for row in v]})
    counts = [[n, k, int(L.ref_scenario_count(n, k))] for n, k in
              [(32, 8), (4, 4), (2, 1), (6, 2), (64, 16), (256, 2), (1000, 500), (60, 30), (5, 7)]]
    return {"sample_vectors": res, "enumerate_vectors": enum, "scenario_count": counts}


def survivors_section():
    """Per-(trial, config) survivor minima from sample_vectors + stage_survivors."""
    L = ref_lib()
    res = []
    for prof, n, k, trials in [("lm_1p5b", 32, 3, 200), ("lm_1p5b", 64, 9, 100), ("toy_six_instance", 6, 2, 15),
                               ("lm_1p5b", 256, 24, 40), ("lm_6p7b", 128, 5, 60)]:
        w = PROFILES[prof]
        cfgs = cfgs_of(w, n)
        seed = int(L.ref_mix_seed(L.ref_mix_seed(0x5EED, n), k))
        buf = (C.c_uint8 * (trials * n))()
        assert L.ref_sample_vectors(n, k, trials, seed, buf) == 0
        m = np.zeros((len(cfgs), trials), dtype=np.uint16)
        for ci, c in enumerate(cfgs):
            out = (C.c_uint16 * trials)()
            L.ref_tally(buf, trials, n, c.pipelines, c.stages, out)
            m[ci] = np.array(out[:], dtype=np.uint16)
        res.append({"profile": prof, "n": n, "k": k, "trials": trials, "seed": seed,
                    "configs": [[c.pipelines, c.stages] for c in cfgs], "m": m.T.tolist()})
    return res


def histogram_section():
    res = []
    cases = [
        ("lm_1p5b", 10000, [(32, 3, [(4, 7), (3, 8), (1, 32), (2, 16), (4, 8)])]),
        ("lm_1p5b", 1000, [(64, 9, None), (128, 2, None), (256, 8, [(36, 7), (1, 256), (5, 50), (17, 15)]),
                           (256, 40, [(36, 7), (10, 25), (2, 100)]), (33, 33, [(4, 8)]), (40, 39, [(5, 8)])]),
        ("lm_6p7b", 3000, [(128, 5, None), (64, 1, None)]),
        ("toy_six_instance", 200, [(6, 2, None), (6, 1, None), (6, 6, None)]),
        ("resnet152", 2000, [(64, 12, [(64, 1), (32, 2), (21, 3), (1, 64), (7, 9)])]),
    ]
    for prof, trials, items in cases:
        w = PROFILES[prof]
        opt = PlannerOptions(mc_trials=trials)
        rp = RefPlanner(w, CostTable(), opt)
        for n, k, cl in items:
            cfgs = cfgs_of(w, n) if cl is None else [ParallelConfig(*c) for c in cl]
            for c in cfgs:
                h = rp.survivor_hist(c, n, k)
                res.append({"profile": prof, "mc_trials": trials, "n": n, "k": k,
                            "cfg": [c.pipelines, c.stages], "hist": [H(x) for x in h]})
    return res


def phi_section():
    res = []
    for prof, trials, cases in [
        ("lm_1p5b", 10000, [((4, 7), (4, 7), 32, 29), ((4, 7), (3, 8), 32, 29), (None, (3, 8), 0, 29),
                            ((4, 8), None, 32, 29), ((4, 8), (4, 8), 32, 40), ((4, 8), (5, 8), 32, 40),
                            ((3, 8), (2, 8), 24, 16), ((1, 32), (1, 7), 32, 7)]),
        ("toy_six_instance", 1000, [((2, 3), (2, 3), 6, 6), ((2, 2), (3, 2), 4, 6), ((2, 3), (1, 1), 6, 6),
                                    ((2, 3), (4, 2), 6, 6), ((3, 2), (2, 2), 6, 4), ((2, 3), (1, 2), 6, 2)]),
        ("lm_1p5b", 500, [((36, 7), (30, 7), 256, 216), ((20, 12), (18, 12), 256, 216),
                          ((5, 50), (4, 50), 256, 200), ((36, 7), (1, 216), 256, 216)]),
    ]:
        w = PROFILES[prof]
        for strict in (False, True):
            rp = RefPlanner(w, CostTable(), PlannerOptions(mc_trials=trials, strict_conditional=strict))
            for pv, nx, a, b in cases:
                p = None if pv is None else ParallelConfig(*pv)
                q = None if nx is None else ParallelConfig(*nx)
                c, m = rp.phi(p, q, a, b)
                res.append({"profile": prof, "mc_trials": trials, "strict": strict, "prev": pv, "next": nx,
                            "n_now": a, "n_next": b, "committed": H(c), "mig": H(m)})
    return res


def plan_section():
    L = ref_lib()
    res = []

    def add(prof, opt, current, n_seq, tag):
        w = PROFILES[prof]
        rp = RefPlanner(w, CostTable(), opt)
        plan = rp.dp_optimize(current, n_seq)
        seq = [s.config for s in plan]
        val = rp.sequence_value(current, seq, n_seq)
        res.append({"tag": tag, "profile": prof, "mc_trials": opt.mc_trials, "exact_cap": opt.exact_cap,
                    "strict": opt.strict_conditional,
                    "current": None if current is None else [current.pipelines, current.stages],
                    "n_seq": list(n_seq),
                    "plan": [[s.interval_index, None if s.config is None else [s.config.pipelines, s.config.stages],
                              H(s.expected_committed), H(s.expected_mig_cost_s)] for s in plan],
                    "value": H(val)})

    ka = [32, 28, 28, 26, 29, 26, 26, 21, 23, 23, 21, 25, 22]
    add("lm_1p5b", PlannerOptions(mc_trials=10000), ParallelConfig(4, 8), ka, "known_answer")
    add("lm_1p5b", PlannerOptions(mc_trials=10000, strict_conditional=True), ParallelConfig(4, 8), ka, "strict")
    add("lm_1p5b", PlannerOptions(mc_trials=10000), None, ka, "from_suspended")
    add("toy_six_instance", PlannerOptions(exact_cap=100000), ParallelConfig(2, 3), [6, 6, 4, 4], "fig_drop")
    add("toy_six_instance", PlannerOptions(exact_cap=100000), ParallelConfig(2, 2), [4, 1, 4], "suspend")
    # synthetic traces (gen_synthetic, trace.cpp:80-180)
    for seed in (1, 2, 3):
        buf = (C.c_int * 64)()
        ln = L.ref_gen_synthetic(seed, 32, 60, 9, 8, 1, 4, buf, 64)
        counts = list(buf[:ln])
        ns = counts[10:23]
        cur_c = (C.c_int * 2)()
        p, keep = lm_1p5b().to_c()
        cur = ParallelConfig(cur_c[0], cur_c[1]) if L.ref_reactive_plan(C.byref(p), ns[0], cur_c) else None
        add("lm_1p5b", PlannerOptions(mc_trials=2000), cur, ns, f"synthetic_{seed}")
    # larger N: MC branch with modest trials
    add("lm_1p5b", PlannerOptions(mc_trials=500), ParallelConfig(8, 8),
        [64, 60, 60, 57, 62, 56, 56, 50], "n64")
    add("lm_6p7b", PlannerOptions(mc_trials=300), ParallelConfig(6, 21),
        [128, 120, 121, 110, 118, 104, 104, 96], "n128_gpt3")
    add("lm_1p5b", PlannerOptions(mc_trials=100), ParallelConfig(36, 7),
        [256, 224, 224, 208, 232, 208], "n256")
    add("resnet152", PlannerOptions(mc_trials=400), ParallelConfig(64, 1),
        [64, 52, 52, 60, 44, 48, 40], "resnet_dp")
    return res


def random_dp_section():
    """DP on random small instances, mirroring test_optimizer.cpp:107-131 (N <= 8)."""
    rng = np.random.default_rng(161803)
    res = []
    for trial in range(60):
        min_depth = int(rng.integers(1, 4))
        w = toy_six_instance()
        w.pipeline_rates = {}
        w.compute_per_microbatch_s = float(0.05 + rng.random() * 2.0)
        w.param_bytes = float(rng.random() * 4e9)
        w.activation_bytes = float(rng.random() * 1e7)
        w.microbatch_size = int(1 + rng.integers(0, 4))
        w.minibatch_size = w.microbatch_size * int(1 + rng.integers(0, 32))
        w.device_memory_bytes = 16.0
        w.memory_fixed_bytes = 0.0
        w.memory_per_stage_bytes = 16.0 * min_depth
        w.alpha_s = float(rng.random() * 0.01)
        w.beta_s_per_byte = float(rng.random() * 2e-9)
        costs = CostTable(*[float(x) for x in rng.random(6) * np.array([1, 10, 10, 10, 10, 20])])
        opt = PlannerOptions(exact_cap=int(rng.choice([0, 20, 100000])), mc_trials=int(rng.integers(1, 300)),
                             interval_s=float(rng.choice([10.0, 60.0])))
        horizon = int(1 + rng.integers(0, 4))
        n_seq = [int(x) for x in rng.integers(0, 9, horizon + 1)]
        starts = cfgs_of(w, n_seq[0])
        current = starts[int(rng.integers(0, len(starts)))] if starts else None
        rp = RefPlanner(w, costs, opt)
        plan = rp.dp_optimize(current, n_seq)
        res.append({"profile": w.__dict__, "costs": costs.__dict__, "options": opt.__dict__,
                    "current": None if current is None else [current.pipelines, current.stages],
                    "n_seq": n_seq,
                    "plan": [[s.interval_index, None if s.config is None else [s.config.pipelines, s.config.stages],
                              H(s.expected_committed), H(s.expected_mig_cost_s)] for s in plan]})
    return res


def tables_section():
    L = ref_lib()
    res = {"throughput": [], "configs": [], "reactive": [], "transition": [], "liveput": []}
    for prof, w in PROFILES.items():
        p, keep = w.to_c()
        for n in (1, 6, 7, 20, 32, 64, 128, 256):
            cs = cfgs_of(w, n)
            res["configs"].append({"profile": prof, "n": n, "configs": [[c.pipelines, c.stages] for c in cs]})
            r = (C.c_int * 2)()
            ok = L.ref_reactive_plan(C.byref(p), n, r)
            res["reactive"].append({"profile": prof, "n": n, "cfg": [r[0], r[1]] if ok else None})
        for d, s in [(1, 1), (2, 3), (3, 2), (4, 7), (36, 7), (1, 256), (64, 1), (7, 9), (5, 20), (2, 2), (0, 3)]:
            res["throughput"].append({"profile": prof, "cfg": [d, s], "value": H(L.ref_throughput(C.byref(p), d, s))})
    w = lm_1p5b()
    p, keep = w.to_c()
    c = CostTable().to_c()
    out = (C.c_double * 2)()
    for m, sd, sp, td, tp, fresh in [(0, 4, 7, 4, 7, 0), (3, 4, 7, 4, 7, 0), (4, 4, 7, 4, 7, 0), (4, 4, 7, 5, 7, 2),
                                     (2, 4, 7, 8, 7, 1), (3, 4, 7, 3, 8, 0), (1, 4, 8, 4, 8, 3), (4, 4, 8, 3, 8, 0)]:
        kind = L.ref_transition_outcome_min(m, sd, sp, td, tp, fresh, C.byref(p), C.byref(c), out)
        res["transition"].append({"args": [m, sd, sp, td, tp, fresh], "kind": kind, "cost": H(out[0]),
                                  "rollback": int(out[1])})
    lv = C.c_double()
    seed_nk = int(L.ref_mix_seed(L.ref_mix_seed(0x5EED, 32), 3))
    for (d, s), n, k, exact, trials, seed in [((4, 7), 32, 3, 0, 10000, seed_nk), ((2, 3), 6, 2, 1, 0, 0),
                                              ((3, 2), 6, 2, 1, 0, 0), ((3, 2), 6, 2, 0, 10000, 9),
                                              ((36, 7), 256, 8, 0, 2000, 5), ((1, 7), 8, 3, 1, 0, 0)]:
        prof = "toy_six_instance" if n == 6 else "lm_1p5b"
        pp, kk = PROFILES[prof].to_c()
        assert L.ref_expected_liveput(C.byref(pp), d, s, n, k, exact, trials, seed, C.byref(lv)) == 0
        res["liveput"].append({"profile": prof, "cfg": [d, s], "n": n, "k": k, "exact": exact, "trials": trials,
                               "seed": seed, "value": H(lv.value)})
    return res


def main():
    sections = {
        "rng": rng_section(),
        "scenarios": scenarios_section(),
        "survivors": survivors_section(),
        "histograms": histogram_section(),
        "phi": phi_section(),
        "plans": plan_section(),
        "random_dp": random_dp_section(),
        "tables": tables_section(),
    }
    for name, data in sections.items():
        (OUT / f"{name}.json").write_text(json.dumps(data, separators=(",", ":")))
        print(name, (OUT / f"{name}.json").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
