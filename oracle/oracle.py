"""CPU ORACLE bindings — test infrastructure only (the checker, never the product).

Two libraries:
  * liboracle.so           — oracle/liveput_oracle.c, the C restatement of the
                             reference hot path (always buildable: gcc).
  * _ref/libspotsim_ref.so — the UNMODIFIED reference (spotsim) compiled from
                             /root/reference by oracle/Makefile (`make ref`),
                             wrapped by oracle/ref_shim.cpp.  Built in the
                             dev container; the .so travels to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path
from typing import List, Optional, Sequence, Tuple

import numpy as np

from paper_2403_14097_b200 import _abi
from paper_2403_14097_b200.model import (CostTable, ParallelConfig, PlannerOptions, PlanStep,
                                         WorkloadProfile)

ORACLE_DIR = Path(__file__).resolve().parent
ORACLE_LIB = ORACLE_DIR / "liboracle.so"
REF_LIB = ORACLE_DIR / "_ref" / "libspotsim_ref.so"
REF_SRC = Path("/root/reference/proj/core")

_P = C.POINTER
_oracle = None
_ref = None


def build_oracle(ref: bool = True) -> None:
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "liboracle.so"], check=True)
    if ref and REF_SRC.exists():
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "ref"], check=True)


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not ORACLE_LIB.exists():
            build_oracle(ref=False)
        l = C.CDLL(str(ORACLE_LIB))
        prof, costs, opts = _P(_abi.lp_profile), _P(_abi.lp_costs), _P(_abi.lp_options)
        sig = {
            "or_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "or_splitmix_next": (C.c_uint64, [_P(C.c_uint64)]),
            "or_sample_distinct": (None, [C.c_int, C.c_int, C.c_uint64, _P(C.c_int)]),
            "or_scenario_count": (C.c_uint64, [C.c_int, C.c_int]),
            "or_depth_feasible": (C.c_int, [prof, C.c_int]),
            "or_throughput": (C.c_double, [prof, C.c_int, C.c_int]),
            "or_enumerate_configs": (C.c_int, [prof, C.c_int, _P(C.c_int), C.c_int]),
            "or_reactive_plan": (C.c_int, [prof, C.c_int, _P(C.c_int)]),
            "or_transition_cost": (C.c_double, [C.c_int] * 6 + [prof, costs, _P(C.c_int), _P(C.c_int)]),
            "or_resume_cost": (C.c_double, [C.c_int, prof, costs]),
            "or_scenarios": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, _P(C.c_int)]),
            "or_ensemble_counts": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, _P(C.c_int),
                                             C.c_int, _P(C.c_uint64), C.c_int, _P(C.c_uint64), C.c_int]),
            "or_ensemble_counts_range": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, _P(C.c_int),
                                                   C.c_int, _P(C.c_uint64), C.c_int, _P(C.c_uint64), C.c_int,
                                                   C.c_longlong, C.c_longlong]),
            "or_planner_new": (C.c_void_p, [prof, costs, opts, C.c_int]),
            "or_planner_free": (None, [C.c_void_p]),
            "or_planner_set_cache": (None, [C.c_void_p, C.c_int]),
            "or_last_error": (C.c_char_p, []),
            "or_survivor_counts": (C.c_int, [C.c_void_p] + [C.c_int] * 4 + [_P(C.c_uint64), _P(C.c_uint64)]),
            "or_phi": (C.c_int, [C.c_void_p] + [C.c_int] * 6 + [_P(C.c_double)]),
            "or_dp_optimize": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _P(C.c_int), C.c_int, _P(C.c_int),
                                         _P(C.c_double), _P(C.c_double)]),
            "or_sequence_value": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _P(C.c_int), _P(C.c_int), C.c_int,
                                            _P(C.c_double)]),
            "or_liveput": (C.c_int, [C.c_void_p] + [C.c_int] * 4 + [_P(C.c_double)]),
        }
        for k, (r, a) in sig.items():
            f = getattr(l, k)
            f.restype, f.argtypes = r, a
        _oracle = l
    return _oracle


def ref_available() -> bool:
    return REF_LIB.exists() or REF_SRC.exists()


def ref_lib():
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            if not REF_SRC.exists():
                raise FileNotFoundError("reference library not built and /root/reference absent")
            build_oracle(ref=True)
        l = C.CDLL(str(REF_LIB))
        prof, costs, opts = _P(_abi.lp_profile), _P(_abi.lp_costs), _P(_abi.lp_options)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_planner_new": (C.c_void_p, [prof, costs, opts]),
            "ref_planner_free": (None, [C.c_void_p]),
            "ref_planner_cache_size": (C.c_size_t, [C.c_void_p]),
            "ref_phi": (C.c_int, [C.c_void_p] + [C.c_int] * 6 + [_P(C.c_double)]),
            "ref_dp_optimize": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _P(C.c_int), C.c_int, _P(C.c_int),
                                          _P(C.c_double)]),
            "ref_sequence_value": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _P(C.c_int), _P(C.c_int), C.c_int,
                                             _P(C.c_double)]),
            "ref_survivor_hist": (C.c_int, [C.c_void_p] + [C.c_int] * 4 + [_P(C.c_double)]),
            "ref_scenario_count": (C.c_uint64, [C.c_int, C.c_int]),
            "ref_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "ref_rng_draws": (None, [C.c_uint64, C.c_int, _P(C.c_uint64)]),
            "ref_sample_distinct": (C.c_int, [C.c_int, C.c_int, C.c_uint64, _P(C.c_int)]),
            "ref_sample_vectors": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, _P(C.c_uint8)]),
            "ref_enumerate_vectors": (C.c_longlong, [C.c_int, C.c_int, _P(C.c_uint8), C.c_longlong]),
            "ref_tally": (None, [_P(C.c_uint8), C.c_int, C.c_int, C.c_int, C.c_int, _P(C.c_uint16)]),
            "ref_surviving_pipelines": (C.c_int, [_P(C.c_uint8), C.c_int, C.c_int, C.c_int, C.c_int]),
            "ref_throughput": (C.c_double, [prof, C.c_int, C.c_int]),
            "ref_depth_feasible": (C.c_int, [prof, C.c_int]),
            "ref_enumerate_configs": (C.c_int, [prof, C.c_int, _P(C.c_int), C.c_int]),
            "ref_reactive_plan": (C.c_int, [prof, C.c_int, _P(C.c_int)]),
            "ref_expected_liveput": (C.c_int, [prof] + [C.c_int] * 6 + [C.c_uint64, _P(C.c_double)]),
            "ref_transition_outcome_min": (C.c_int, [C.c_int] * 6 + [prof, costs, _P(C.c_double)]),
            "ref_resume_cost": (C.c_double, [C.c_int, C.c_int, prof, costs]),
            "ref_predict": (C.c_int, [_P(C.c_int), C.c_int, _P(C.c_int), _P(C.c_double), C.c_int, _P(C.c_int)]),
            "ref_eval_l1": (C.c_double, [_P(C.c_int), _P(C.c_int), C.c_int]),
            "ref_simulate": (C.c_int, [_P(C.c_int), C.c_int, C.c_double, C.c_int, prof, C.c_double, C.c_double, costs,
                                       opts, _P(C.c_int), _P(C.c_double), C.c_uint64, C.c_int, _P(C.c_double),
                                       _P(C.c_int), _P(C.c_longlong), _P(C.c_double)]),
            "ref_plan_migration": (C.c_int, [C.c_int] * 3 + [_P(C.c_uint8), C.c_int, C.c_int, C.c_int, prof, costs,
                                             _P(C.c_int), _P(C.c_int), C.c_int, _P(C.c_double)]),
            "ref_gen_synthetic": (C.c_int, [C.c_uint64] + [C.c_int] * 6 + [_P(C.c_int), C.c_int]),
            "ref_bench_histograms": (C.c_double, [prof, costs, opts, _P(C.c_int), _P(C.c_int), C.c_int, C.c_int,
                                                  _P(C.c_ulonglong)]),
            "ref_bench_replan": (C.c_double, [prof, costs, opts, C.c_int, C.c_int, _P(C.c_int), C.c_int]),
        }
        for k, (r, a) in sig.items():
            f = getattr(l, k)
            f.restype, f.argtypes = r, a
        _ref = l
    return _ref


def _ints(seq):
    arr = (C.c_int * max(len(seq), 1))(*seq)
    return arr


def _cfg_pair(cfg: Optional[ParallelConfig]) -> Tuple[int, int]:
    return (0, 0) if cfg is None else (cfg.pipelines, cfg.stages)


class _PlannerBase:
    def __init__(self, w: WorkloadProfile, costs: CostTable, opt: PlannerOptions):
        self.w, self.costs, self.opt = w, costs, opt
        self._p, self._keep = w.to_c()
        self._c = costs.to_c()
        self._o = opt.to_c()


class RefPlanner(_PlannerBase):
    """spotsim::Planner itself (compiled reference)."""

    def __init__(self, w, costs=None, opt=None):
        super().__init__(w, costs or CostTable(), opt or PlannerOptions())
        self.L = ref_lib()
        self.h = self.L.ref_planner_new(C.byref(self._p), C.byref(self._c), C.byref(self._o))

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_planner_free(self.h)
            self.h = None

    def _chk(self, rc):
        if rc != 0:
            raise ValueError(self.L.ref_last_error().decode())

    def phi(self, prev, nxt, n_now, n_next):
        out = (C.c_double * 2)()
        self._chk(self.L.ref_phi(self.h, *_cfg_pair(prev), *_cfg_pair(nxt), n_now, n_next, out))
        return out[0], out[1]

    def dp_optimize(self, current, n_seq) -> List[PlanStep]:
        h = len(n_seq) - 1
        cfg = (C.c_int * max(2 * h, 2))()
        val = (C.c_double * max(2 * h, 2))()
        self._chk(self.L.ref_dp_optimize(self.h, *_cfg_pair(current), _ints(n_seq), len(n_seq), cfg, val))
        return [PlanStep(j + 1, None if cfg[2 * j] <= 0 else ParallelConfig(cfg[2 * j], cfg[2 * j + 1]),
                         val[2 * j], val[2 * j + 1]) for j in range(h)]

    def sequence_value(self, current, seq, n_seq):
        flat = []
        for c in seq:
            flat += list(_cfg_pair(c))
        out = C.c_double()
        self._chk(self.L.ref_sequence_value(self.h, *_cfg_pair(current), _ints(flat), _ints(n_seq),
                                            len(n_seq), C.byref(out)))
        return out.value

    def survivor_hist(self, cfg: ParallelConfig, n_now, n_minus) -> np.ndarray:
        out = (C.c_double * (cfg.pipelines + 1))()
        self._chk(self.L.ref_survivor_hist(self.h, cfg.pipelines, cfg.stages, n_now, n_minus, out))
        return np.array(out[:], dtype=np.float64)


class OraclePlanner(_PlannerBase):
    """The C restatement (cache-free) — used where the reference is absent or aliases."""

    def __init__(self, w, costs=None, opt=None, threads: int = 0, cache: bool = False):
        super().__init__(w, costs or CostTable(), opt or PlannerOptions())
        self.L = oracle_lib()
        threads = threads or min(8, os.cpu_count() or 1)
        self.h = self.L.or_planner_new(C.byref(self._p), C.byref(self._c), C.byref(self._o), threads)
        if cache:  # memo of full-level ensembles for long replays (identical results)
            self.L.or_planner_set_cache(self.h, 1)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.or_planner_free(self.h)
            self.h = None

    def _chk(self, rc):
        if rc != 0:
            raise ValueError(self.L.or_last_error().decode())

    def phi(self, prev, nxt, n_now, n_next):
        out = (C.c_double * 2)()
        self._chk(self.L.or_phi(self.h, *_cfg_pair(prev), *_cfg_pair(nxt), n_now, n_next, out))
        return out[0], out[1]

    def dp_optimize(self, current, n_seq, with_value=False):
        h = len(n_seq) - 1
        cfg = (C.c_int * max(2 * h, 2))()
        val = (C.c_double * max(2 * h, 2))()
        fv = C.c_double()
        self._chk(self.L.or_dp_optimize(self.h, *_cfg_pair(current), _ints(n_seq), len(n_seq), cfg, val,
                                        C.byref(fv)))
        plan = [PlanStep(j + 1, None if cfg[2 * j] <= 0 else ParallelConfig(cfg[2 * j], cfg[2 * j + 1]),
                         val[2 * j], val[2 * j + 1]) for j in range(h)]
        return (plan, fv.value) if with_value else plan

    def sequence_value(self, current, seq, n_seq):
        flat = []
        for c in seq:
            flat += list(_cfg_pair(c))
        out = C.c_double()
        self._chk(self.L.or_sequence_value(self.h, *_cfg_pair(current), _ints(flat), _ints(n_seq),
                                           len(n_seq), C.byref(out)))
        return out.value

    def survivor_counts(self, cfg: ParallelConfig, n_now, n_minus):
        out = (C.c_uint64 * (cfg.pipelines + 1))()
        tot = C.c_uint64()
        self._chk(self.L.or_survivor_counts(self.h, cfg.pipelines, cfg.stages, n_now, n_minus, out,
                                            C.byref(tot)))
        return np.array(out[:], dtype=np.uint64), tot.value

    def liveput(self, cfg: ParallelConfig, n_now, n_minus):
        out = C.c_double()
        self._chk(self.L.or_liveput(self.h, cfg.pipelines, cfg.stages, n_now, n_minus, C.byref(out)))
        return out.value


def oracle_scenarios(n, k, exact, trials, seed) -> np.ndarray:
    L = oracle_lib()
    out = (C.c_int * max(trials * k, 1))()
    if L.or_scenarios(n, k, int(exact), trials, seed, out) != 0:
        raise ValueError(L.or_last_error().decode())
    return np.array(out[: trials * k], dtype=np.int64).reshape(trials, k)


def oracle_ensemble_counts(n, k, exact, trials, seed, cfgs: Sequence[ParallelConfig], threads=0):
    L = oracle_lib()
    stride = max(c.pipelines for c in cfgs) + 1
    flat = []
    for c in cfgs:
        flat += [c.pipelines, c.stages]
    out = (C.c_uint64 * (len(cfgs) * stride))()
    tot = C.c_uint64()
    threads = threads or min(8, os.cpu_count() or 1)
    if L.or_ensemble_counts(n, k, int(exact), trials, seed, _ints(flat), len(cfgs), out, stride,
                            C.byref(tot), threads) != 0:
        raise ValueError(L.or_last_error().decode())
    return np.array(out[:], dtype=np.uint64).reshape(len(cfgs), stride), tot.value


def oracle_ensemble_counts_range(n, k, exact, trials, seed, cfgs: Sequence[ParallelConfig], r0, r1, threads=0):
    """Partial ensemble over scenario ranks [r0, r1) (the multi-rank trial split)."""
    L = oracle_lib()
    stride = max(c.pipelines for c in cfgs) + 1
    flat = []
    for c in cfgs:
        flat += [c.pipelines, c.stages]
    out = (C.c_uint64 * (len(cfgs) * stride))()
    tot = C.c_uint64()
    threads = threads or min(8, os.cpu_count() or 1)
    if L.or_ensemble_counts_range(n, k, int(exact), trials, seed, _ints(flat), len(cfgs), out, stride,
                                  C.byref(tot), threads, r0, r1) != 0:
        raise ValueError(L.or_last_error().decode())
    return np.array(out[:], dtype=np.uint64).reshape(len(cfgs), stride), tot.value


def oracle_configs(w: WorkloadProfile, n: int) -> List[ParallelConfig]:
    L = oracle_lib()
    p, keep = w.to_c()
    cnt = L.or_enumerate_configs(C.byref(p), n, None, 0)
    out = (C.c_int * max(2 * cnt, 2))()
    L.or_enumerate_configs(C.byref(p), n, out, cnt)
    return [ParallelConfig(out[2 * i], out[2 * i + 1]) for i in range(cnt)]


def oracle_throughput(w: WorkloadProfile, cfg: ParallelConfig) -> float:
    p, keep = w.to_c()
    return oracle_lib().or_throughput(C.byref(p), cfg.pipelines, cfg.stages)


def oracle_reactive(w: WorkloadProfile, n: int) -> Optional[ParallelConfig]:
    p, keep = w.to_c()
    out = (C.c_int * 2)()
    return ParallelConfig(out[0], out[1]) if oracle_lib().or_reactive_plan(C.byref(p), n, out) else None


def mix_seed(a, b):
    return oracle_lib().or_mix_seed(a, b)


def planner_seed(mc_seed, n, k):
    """optimizer.cpp:88-89: mix_seed(mix_seed(mc_seed, n), k)."""
    return mix_seed(mix_seed(mc_seed, n), k)


def ref_plan_migration(w: WorkloadProfile, costs: CostTable, source: ParallelConfig, spares: int, v,
                       target: ParallelConfig):
    """The reference's plan_migration through oracle/_ref (test infrastructure).
    Returns ("ok", kind, rounds, moves, est_cost, cost_fresh) or ("rollback",) /
    ("invalid",)."""
    l = ref_lib()
    p, keep = w.to_c()
    c = costs.to_c()
    n = len(v)
    vb = (C.c_uint8 * max(n, 1))(*[1 if x else 0 for x in v])
    info = (C.c_int * 3)()
    cap = max(n, 1)
    mv = (C.c_int * (6 * cap))()
    cost = (C.c_double * 2)()
    rc = l.ref_plan_migration(source.pipelines, source.stages, spares, vb, n, target.pipelines, target.stages,
                              C.byref(p), C.byref(c), info, mv, cap, cost)
    if rc == 1:
        return ("rollback",)
    if rc == 2:
        return ("invalid",)
    moves = [tuple(mv[6 * i: 6 * i + 6]) for i in range(min(info[2], cap))]
    return ("ok", info[0], info[1], moves, cost[0], cost[1])


def ref_transition_outcome(w: WorkloadProfile, costs: CostTable, m, sd, sp, td, tp, fresh):
    """The reference's transition_outcome_min: (cost_s, kind name, rollback)."""
    l = ref_lib()
    p, keep = w.to_c()
    c = costs.to_c()
    out = (C.c_double * 2)()
    kind = l.ref_transition_outcome_min(m, sd, sp, td, tp, fresh, C.byref(p), C.byref(c), out)
    names = {0: "none", 1: "intra_stage", 2: "inter_stage", 3: "pipeline"}
    return out[0], names[kind], bool(out[1])


def ref_predict(history, cfg, method: int):
    """The reference's predict() through oracle/_ref; None on invalid_argument."""
    l = ref_lib()
    h = (C.c_int * max(len(history), 1))(*history)
    ci = (C.c_int * 7)(cfg.history_len, cfg.lookahead, cfg.capacity, cfg.floor, cfg.max_step,
                       cfg.reset_threshold, cfg.moving_avg_window)
    cd = (C.c_double * 2)(cfg.exp_smooth_factor, cfg.steep_decay)
    out = (C.c_int * max(cfg.lookahead, 1))()
    if l.ref_predict(h, len(history), ci, cd, method, out) != 0:
        return None
    return list(out[: cfg.lookahead])


def ref_eval_l1(pred, actual):
    l = ref_lib()
    a = (C.c_int * max(len(pred), 1))(*pred)
    b = (C.c_int * max(len(actual), 1))(*actual)
    return l.ref_eval_l1(a, b, len(pred))


def ref_gen_synthetic(seed, cap, length, loss_events, gain_events, min_step, max_step):
    l = ref_lib()
    out = (C.c_int * (length + 8))()
    n = l.ref_gen_synthetic(seed, cap, length, loss_events, gain_events, min_step, max_step, out, length + 8)
    return list(out[:n])


def ref_simulate(counts, w, pol, seed, opt, costs, interval_s=60.0, capacity=0, epoch_samples=0, spot=0.0,
                 ondemand=0.0):
    """The reference's run() through oracle/_ref; same dict layout as
    paper_2403_14097_b200.planner.simulate."""
    import math
    l = ref_lib()
    p, keep = w.to_c()
    c = costs.to_c()
    o = opt.to_c()
    n = len(counts)
    cnt = (C.c_int * max(n, 1))(*counts)
    pi = (C.c_int * 6)(pol.kind, pol.lookahead, pol.method, pol.history, pol.ckpt_period_intervals,
                       pol.redundancy_fixed_stages)
    pd = (C.c_double * 4)(pol.ckpt_save_cost_s, pol.ckpt_restore_cost_s, pol.ckpt_restart_cost_s,
                          pol.redundancy_slowdown)
    rd = (C.c_double * 12)()
    ri = (C.c_int * 4)()
    li = (C.c_longlong * (7 * max(n, 1)))()
    ld = (C.c_double * (6 * max(n, 1)))()
    rc = l.ref_simulate(cnt, n, interval_s, capacity, C.byref(p), spot, ondemand, C.byref(c), C.byref(o), pi, pd,
                        seed, epoch_samples, rd, ri, li, ld)
    if rc != 0:
        raise ValueError(l.ref_last_error().decode())
    led = lambda a: {"effective_s": a[0], "migration_s": a[1], "checkpoint_s": a[2], "wasted_rollback_s": a[3],
                     "idle_s": a[4]}
    report = {"seed": seed, "committed_samples": int(rd[0]), "wall_time_s": rd[1], "ledger": led(rd[2:7]),
              "instance_seconds": rd[7], "instance_hours": rd[8], "spot_cost": rd[9], "ondemand_cost": rd[10],
              "cost_per_sample": None if math.isnan(rd[11]) else rd[11], "epochs_completed": ri[0],
              "rollback_events": ri[1], "suspended_intervals": ri[2], "sample_accounting_ok": bool(ri[3])}
    names = ["none", "intra_stage", "inter_stage", "pipeline"]
    ivs = [{"interval": li[7 * i], "available": li[7 * i + 1], "pipelines": li[7 * i + 2], "stages": li[7 * i + 3],
            "throughput": ld[6 * i], "committed": li[7 * i + 4], "rolled_back": li[7 * i + 5],
            "migration": names[li[7 * i + 6]], "ledger": led(ld[6 * i + 1: 6 * i + 6])} for i in range(n)]
    return report, ivs
