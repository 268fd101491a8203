"""Python mirror of ``spotsim::Planner`` (optimizer.hpp:41-92) over the C ABI.

Same names, argument meaning and error behaviour as the reference: ``None``
is the suspended configuration (std::nullopt), bad arguments raise
ValueError (the reference's std::invalid_argument).  Every computation runs
in libliveput.so on the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from .model import (CostTable, ParallelConfig, PlannerOptions, PlanStep, WorkloadProfile,
                    cfg_from_c, cfg_to_c)


@dataclass
class PhiValue:
    committed: float = 0.0
    mig_cost_s: float = 0.0


@dataclass
class LiveputRow:
    interval: int
    config: ParallelConfig
    liveput: float


class Planner:
    """Availability-aware configuration planner (liveput DP) on one B200."""

    def __init__(self, w: WorkloadProfile, costs: Optional[CostTable] = None,
                 opt: Optional[PlannerOptions] = None, device: int = 0):
        self._lib = _abi.lib()
        self.w = w
        self.costs = costs or CostTable()
        self.opt = opt or PlannerOptions()
        self._prof, self._keep = w.to_c()
        self._c = self.costs.to_c()
        self._o = self.opt.to_c()
        h = C.c_void_p()
        _abi.check(self._lib.lp_create(C.byref(self._prof), C.byref(self._c), C.byref(self._o),
                                       device, C.byref(h)))
        self._h = h
        self.last_liveput: List[LiveputRow] = []

    def close(self):
        if getattr(self, "_h", None):
            self._lib.lp_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- reference API -------------------------------------------------
    def workload(self) -> WorkloadProfile:
        return self.w

    def options(self) -> PlannerOptions:
        return self.opt

    def phi(self, prev: Optional[ParallelConfig], nxt: Optional[ParallelConfig], n_now: int,
            n_next: int) -> PhiValue:
        c, m = C.c_double(), C.c_double()
        _abi.check(self._lib.lp_phi(self._h, cfg_to_c(prev), cfg_to_c(nxt), n_now, n_next,
                                    C.byref(c), C.byref(m)), self._h)
        return PhiValue(c.value, m.value)

    def dp_optimize(self, current: Optional[ParallelConfig], n_seq: Sequence[int],
                    want_liveput: bool = False) -> List[PlanStep]:
        n = len(n_seq)
        if n < 2:
            raise ValueError("dp_optimize: need at least N_i and N_{i+1}")
        ns = (C.c_int32 * n)(*n_seq)
        out = (_abi.lp_plan_step * (n - 1))()
        cap = 0
        live = None
        rows = C.c_int32(0)
        if want_liveput:
            cap = sum(len(self.configs(x)) for x in n_seq) + 1
            live = (_abi.lp_liveput_row * cap)()
        _abi.check(self._lib.lp_replan(self._h, cfg_to_c(current), ns, n, out, live, cap,
                                       C.byref(rows)), self._h)
        if want_liveput:
            self.last_liveput = [LiveputRow(r.interval, cfg_from_c(r.config), r.liveput)
                                 for r in live[: min(rows.value, cap)]]
        return [PlanStep(s.interval_index, cfg_from_c(s.config), s.expected_committed,
                         s.expected_mig_cost_s) for s in out]

    def sequence_value(self, current: Optional[ParallelConfig],
                       sequence: Sequence[Optional[ParallelConfig]], n_seq: Sequence[int]) -> float:
        if len(sequence) + 1 != len(n_seq):
            raise ValueError("sequence_value: sequence/N length mismatch")
        seq = (_abi.lp_config * max(len(sequence), 1))(*[cfg_to_c(c) for c in sequence])
        ns = (C.c_int32 * len(n_seq))(*n_seq)
        out = C.c_double()
        _abi.check(self._lib.lp_sequence_value(self._h, cfg_to_c(current), seq, ns, len(n_seq),
                                               C.byref(out)), self._h)
        return out.value

    # ---- hot-path internals exposed for parity -------------------------
    def survivor_counts(self, prev: ParallelConfig, n_now: int, n_minus: int) -> Tuple[np.ndarray, int]:
        counts = (C.c_uint64 * (prev.pipelines + 1))()
        tot = C.c_uint64()
        _abi.check(self._lib.lp_survivor_hist(self._h, prev.to_c(), n_now, n_minus, counts,
                                              C.byref(tot)), self._h)
        return np.array(counts[:], dtype=np.uint64), tot.value

    def survivor_histogram(self, prev: ParallelConfig, n_now: int, n_minus: int) -> np.ndarray:
        counts, tot = self.survivor_counts(prev, n_now, n_minus)
        return counts.astype(np.float64) / float(tot)

    def expected_liveput(self, cfg: ParallelConfig, n: int, n_minus: int, exact: bool = True,
                         trials: int = 1000, seed: int = 0) -> float:
        out = C.c_double()
        _abi.check(self._lib.lp_expected_liveput(self._h, cfg.to_c(), n, n_minus, int(exact), trials,
                                                 seed, C.byref(out)), self._h)
        return out.value

    def dump_survivors(self, n: int, n_minus: int, trials: int, seed: int,
                       cfgs: Sequence[ParallelConfig], exact: bool = False) -> np.ndarray:
        arr = (_abi.lp_config * len(cfgs))(*[c.to_c() for c in cfgs])
        out = np.zeros((trials, len(cfgs)), dtype=np.uint16)
        _abi.check(self._lib.lp_dump_survivors(
            self._h, n, n_minus, int(exact), trials, seed, arr, len(cfgs),
            out.ctypes.data_as(C.POINTER(C.c_uint16))), self._h)
        return out

    def dump_scenarios(self, n: int, n_minus: int, trials: int, seed: int) -> np.ndarray:
        out = np.zeros((trials, max(n_minus, 1)), dtype=np.uint16)
        _abi.check(self._lib.lp_dump_scenarios(self._h, n, n_minus, trials, seed,
                                               out.ctypes.data_as(C.POINTER(C.c_uint16))), self._h)
        return out[:, :n_minus]

    # ---- split re-plan for device-resident timing ----------------------
    def prepare(self, current: Optional[ParallelConfig], n_seq: Sequence[int]) -> None:
        ns = (C.c_int32 * len(n_seq))(*n_seq)
        _abi.check(self._lib.lp_prepare(self._h, cfg_to_c(current), ns, len(n_seq)), self._h)

    def execute(self) -> None:
        _abi.check(self._lib.lp_execute(self._h), self._h)

    def fetch(self, horizon: int) -> List[PlanStep]:
        out = (_abi.lp_plan_step * horizon)()
        _abi.check(self._lib.lp_fetch(self._h, out, None, 0, None), self._h)
        return [PlanStep(s.interval_index, cfg_from_c(s.config), s.expected_committed,
                         s.expected_mig_cost_s) for s in out]

    def stats(self) -> _abi.lp_stats:
        st = _abi.lp_stats()
        _abi.check(self._lib.lp_get_stats(self._h, C.byref(st)), self._h)
        return st

    def set_hist_cache(self, enable: bool = True, max_bytes: int = 4 << 30) -> None:
        """Reuse (n, k) ensembles across re-plans, like the reference's hist_cache_."""
        _abi.check(self._lib.lp_set_hist_cache(self._h, int(enable), max_bytes), self._h)

    def precompute(self, pairs) -> None:
        """Offline liveput tables: sample every config of n at each (n, k)."""
        pairs = list(pairs)
        ns = (C.c_int32 * max(len(pairs), 1))(*[p[0] for p in pairs])
        ks = (C.c_int32 * max(len(pairs), 1))(*[p[1] for p in pairs])
        _abi.check(self._lib.lp_precompute(self._h, ns, ks, len(pairs)), self._h)

    def export_tables(self) -> bytes:
        n = C.c_uint64()
        _abi.check(self._lib.lp_cache_export(self._h, None, 0, C.byref(n)), self._h)
        buf = (C.c_uint8 * n.value)()
        _abi.check(self._lib.lp_cache_export(self._h, buf, n.value, C.byref(n)), self._h)
        return bytes(buf)

    def import_tables(self, data: bytes) -> None:
        buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
        _abi.check(self._lib.lp_cache_import(self._h, buf, len(data)), self._h)

    def stream_ptr(self) -> int:
        return self._lib.lp_stream(self._h) or 0

    def comm_init(self, uid: bytes, nranks: int, rank: int) -> None:
        arr = (C.c_uint8 * _abi.LP_NCCL_ID_BYTES).from_buffer_copy(uid)
        _abi.check(self._lib.lp_comm_init(self._h, arr, nranks, rank), self._h)

    def set_shard(self, rank: int, nranks: int) -> None:
        """survivor_counts over trial slice `rank` of an `nranks`-way split
        (parity mode of the multi-GPU decomposition; lp_set_shard)."""
        _abi.check(self._lib.lp_set_shard(self._h, rank, nranks), self._h)

    # ---- host table producers -----------------------------------------
    def configs(self, n: int) -> List[ParallelConfig]:
        return enumerate_configs(n, self.w)


def nccl_unique_id() -> bytes:
    arr = (C.c_uint8 * _abi.LP_NCCL_ID_BYTES)()
    _abi.check(_abi.lib().lp_nccl_unique_id(arr))
    return bytes(arr)


def enumerate_configs(n: int, w: WorkloadProfile) -> List[ParallelConfig]:
    """perf_model.cpp:44-52 (host table producer)."""
    lib = _abi.lib()
    p, keep = w.to_c()
    cnt = lib.lp_enumerate_configs(C.byref(p), n, None, 0)
    out = (_abi.lp_config * max(cnt, 1))()
    lib.lp_enumerate_configs(C.byref(p), n, out, cnt)
    return [ParallelConfig(out[i].pipelines, out[i].stages) for i in range(cnt)]


def throughput(cfg: ParallelConfig, w: WorkloadProfile) -> float:
    p, keep = w.to_c()
    return _abi.lib().lp_throughput(C.byref(p), cfg.to_c())


def reactive_plan(n_now: int, w: WorkloadProfile) -> Optional[ParallelConfig]:
    p, keep = w.to_c()
    out = _abi.lp_config()
    return cfg_from_c(out) if _abi.lib().lp_reactive_plan(C.byref(p), n_now, C.byref(out)) else None


def scenario_count(n: int, k: int) -> int:
    return _abi.lib().lp_scenario_count(n, k)


def mix_seed(a: int, b: int) -> int:
    return _abi.lib().lp_mix_seed(a, b)


# ---- migration planning for a realised scenario ----------
RollbackRequired = _abi.RollbackRequired
MIGRATION_KINDS = {_abi.LP_MIG_NONE: "none", _abi.LP_MIG_INTRA_STAGE: "intra_stage",
                   _abi.LP_MIG_INTER_STAGE: "inter_stage", _abi.LP_MIG_PIPELINE: "pipeline"}


@dataclass
class Move:
    """Move (migration.hpp:29-34); from_* are -1 for a spare instance."""
    instance: int
    from_pipeline: int
    from_stage: int
    to_pipeline: int
    to_stage: int
    transfers_params: bool


@dataclass
class MigrationPlan:
    """MigrationPlan (migration.hpp:36-43)."""
    kind: str
    moves: List[Move]
    source: ParallelConfig
    target: ParallelConfig
    transfer_rounds: int
    est_cost_s: float
    _c: object = None

    def cost(self, w: WorkloadProfile, costs: CostTable, fresh_instances: int = 0) -> float:
        """migration_cost (migration.cpp:219-236)."""
        p, keep = w.to_c()
        c = costs.to_c()
        return _abi.lib().lp_migration_cost(C.byref(p), C.byref(c), C.byref(self._c), fresh_instances)


def plan_migration(source: ParallelConfig, spares: int, v: Sequence[int], target: ParallelConfig,
                   w: WorkloadProfile, costs: CostTable) -> MigrationPlan:
    """plan_migration (migration.cpp:106-217) for topology (source, spares) under
    preemption vector v (1 = preempted).  Raises RollbackRequired when a stage has
    no survivor, ValueError on a size mismatch or too few instances."""
    lib = _abi.lib()
    p, keep = w.to_c()
    c = costs.to_c()
    n = len(v)
    vb = (C.c_uint8 * max(n, 1))(*[1 if x else 0 for x in v])
    out = _abi.lp_migration()
    cap = max(n, 1)
    moves = (_abi.lp_move * cap)()
    _abi.check(lib.lp_plan_migration(C.byref(p), C.byref(c), source.to_c(), spares, vb, n, target.to_c(),
                                     C.byref(out), moves, cap))
    mv = [Move(m.instance, m.from_pipeline, m.from_stage, m.to_pipeline, m.to_stage, bool(m.transfers_params))
          for m in moves[: min(out.n_moves, cap)]]
    return MigrationPlan(MIGRATION_KINDS[out.kind], mv, ParallelConfig(out.source.pipelines, out.source.stages),
                         ParallelConfig(out.target.pipelines, out.target.stages), out.transfer_rounds,
                         out.est_cost_s, out)


def transition_outcome(min_survivor: int, source: ParallelConfig, target: ParallelConfig,
                       fresh_instances: int, w: WorkloadProfile, costs: CostTable) -> Tuple[float, str, bool]:
    """transition_outcome_min (migration.cpp:49-89): (cost_s, kind, rollback)."""
    p, keep = w.to_c()
    c = costs.to_c()
    cost, kind, rb = C.c_double(), C.c_int32(), C.c_int32()
    _abi.check(_abi.lib().lp_transition_outcome(C.byref(p), C.byref(c), min_survivor, source.to_c(),
                                                target.to_c(), fresh_instances, C.byref(cost), C.byref(kind),
                                                C.byref(rb)))
    return cost.value, MIGRATION_KINDS[kind.value], bool(rb.value)


def resume_cost(target: ParallelConfig, w: WorkloadProfile, costs: CostTable) -> float:
    """resume_cost (migration.cpp:100-104)."""
    p, keep = w.to_c()
    c = costs.to_c()
    return _abi.lib().lp_resume_cost(C.byref(p), C.byref(c), target.to_c())


# ---- availability forecasts: the DP's n_seq producer ------
PREDICT_METHODS = {"arima": _abi.LP_PREDICT_ARIMA, "moving_avg": _abi.LP_PREDICT_MOVING_AVG,
                   "exp_smooth": _abi.LP_PREDICT_EXP_SMOOTH, "last_value": _abi.LP_PREDICT_LAST_VALUE}


@dataclass
class ForecastConfig:
    """ForecastConfig (predictor.hpp:8-18)."""
    history_len: int = 12
    lookahead: int = 12
    capacity: int = 0
    floor: int = 0
    max_step: int = 8
    reset_threshold: int = 10
    moving_avg_window: int = 4
    exp_smooth_factor: float = 0.5
    steep_decay: float = 0.7

    def to_c(self) -> _abi.lp_forecast_config:
        return _abi.lp_forecast_config(self.history_len, self.lookahead, self.capacity, self.floor,
                                       self.max_step, self.reset_threshold, self.moving_avg_window, 0,
                                       self.exp_smooth_factor, self.steep_decay)


def _method(m) -> int:
    if isinstance(m, str):
        if m not in PREDICT_METHODS:
            raise ValueError(f"unknown predict method: {m}")
        return PREDICT_METHODS[m]
    return int(m)


def predict(history: Sequence[int], cfg: ForecastConfig, method="arima", device: int = 0) -> List[int]:
    """predict (predictor.cpp:239-274), evaluated on the GPU."""
    h = (C.c_int32 * max(len(history), 1))(*history)
    out = (C.c_int32 * max(cfg.lookahead, 1))()
    c = cfg.to_c()
    _abi.check(_abi.lib().lp_predict(h, len(history), C.byref(c), _method(method), device, out))
    return list(out[: cfg.lookahead])


def predict_windows(counts: Sequence[int], cfg: ForecastConfig, methods=("arima",), device: int = 0):
    """Every sliding window of `spotsim predict` (commands.cpp:267-299) at once:
    returns (preds[window][method] -> list, l1[window][method])."""
    ms = [_method(m) for m in methods]
    n = len(counts)
    nw = max(0, n - cfg.history_len - cfg.lookahead + 1)
    cnt = (C.c_int32 * max(n, 1))(*counts)
    mth = (C.c_int32 * len(ms))(*ms)
    preds = (C.c_int32 * max(nw * len(ms) * cfg.lookahead, 1))()
    l1 = (C.c_double * max(nw * len(ms), 1))()
    got = C.c_int32()
    c = cfg.to_c()
    _abi.check(_abi.lib().lp_predict_windows(cnt, n, C.byref(c), mth, len(ms), device, preds, l1, C.byref(got)))
    I, M = cfg.lookahead, len(ms)
    P = [[list(preds[(w * M + m) * I:(w * M + m + 1) * I]) for m in range(M)] for w in range(got.value)]
    L = [[l1[w * M + m] for m in range(M)] for w in range(got.value)]
    return P, L


def eval_l1(pred: Sequence[int], actual: Sequence[int]) -> float:
    """eval_l1 (predictor.cpp:276-286)."""
    if len(pred) != len(actual):
        raise ValueError("eval_l1: length mismatch")
    n = len(pred)
    a = (C.c_int32 * max(n, 1))(*pred)
    b = (C.c_int32 * max(n, 1))(*actual)
    return _abi.lib().lp_eval_l1(a, b, n)


# ---- the replay driver: the reference simulator's run() ----
POLICIES = {"proactive": _abi.LP_POLICY_PROACTIVE, "ideal": _abi.LP_POLICY_IDEAL,
            "reactive": _abi.LP_POLICY_REACTIVE, "checkpoint": _abi.LP_POLICY_CHECKPOINT,
            "redundancy": _abi.LP_POLICY_REDUNDANCY}
_MIG_NAMES = ["none", "intra_stage", "inter_stage", "pipeline"]


def policy(name: str, **kw) -> _abi.lp_policy:
    """Policy (simulator.hpp:38-75) with the reference's defaults; keyword
    arguments override lp_policy fields (lookahead, method, history,
    ckpt_period_intervals, ckpt_save_cost_s, ..., redundancy_fixed_stages)."""
    if name not in POLICIES:
        raise ValueError(f"unknown policy: {name}")
    p = _abi.lib().lp_policy_defaults(POLICIES[name])
    for k, v in kw.items():
        setattr(p, k, _method(v) if k == "method" else v)
    return p


def _report_dicts(rep, logs, n):
    led = lambda L: {"effective_s": L.effective_s, "migration_s": L.migration_s, "checkpoint_s": L.checkpoint_s,
                     "wasted_rollback_s": L.wasted_rollback_s, "idle_s": L.idle_s}
    report = {"seed": rep.seed, "committed_samples": rep.committed_samples, "wall_time_s": rep.wall_time_s,
              "ledger": led(rep.ledger), "instance_seconds": rep.instance_seconds,
              "instance_hours": rep.instance_hours, "spot_cost": rep.spot_cost, "ondemand_cost": rep.ondemand_cost,
              "cost_per_sample": rep.cost_per_sample if rep.has_cost_per_sample else None,
              "epochs_completed": rep.epochs_completed, "rollback_events": rep.rollback_events,
              "suspended_intervals": rep.suspended_intervals, "sample_accounting_ok": bool(rep.sample_accounting_ok)}
    ivs = [{"interval": L.interval, "available": L.available, "pipelines": L.pipelines, "stages": L.stages,
            "throughput": L.throughput, "committed": L.committed, "rolled_back": L.rolled_back,
            "migration": _MIG_NAMES[L.migration], "ledger": led(L.ledger)} for L in logs[:n]]
    return report, ivs


def simulate_batch(counts: Sequence[int], w: WorkloadProfile, pol: _abi.lp_policy, seeds: Sequence[int],
                   opt: Optional[PlannerOptions] = None, costs: Optional[CostTable] = None, interval_s: float = 60.0,
                   capacity: int = 0, epoch_samples: int = 0, spot_price_per_hour: float = 0.0,
                   ondemand_price_per_hour: float = 0.0, planner: Optional["Planner"] = None, device: int = 0):
    """run() for every seed, planning the trace once (lp_simulate_batch)."""
    lib = _abi.lib()
    p, keep = w.to_c()
    c = (costs or CostTable()).to_c()
    o = (opt or PlannerOptions()).to_c()
    n, m = len(counts), len(seeds)
    cnt = (C.c_int32 * max(n, 1))(*counts)
    sd = (C.c_uint64 * max(m, 1))(*seeds)
    reps = (_abi.lp_sim_report * max(m, 1))()
    logs = (_abi.lp_interval_log * max(n * m, 1))()
    _abi.check(lib.lp_simulate_batch(planner._h if planner else None, C.byref(p), C.byref(c), C.byref(o), device,
                                     cnt, n, interval_s, capacity, C.byref(pol), sd, m, epoch_samples,
                                     spot_price_per_hour, ondemand_price_per_hour, reps, logs))
    return [_report_dicts(reps[q], logs[q * n:(q + 1) * n], n) for q in range(m)]


def simulate(counts: Sequence[int], w: WorkloadProfile, pol: _abi.lp_policy, seed: int,
             opt: Optional[PlannerOptions] = None, costs: Optional[CostTable] = None, interval_s: float = 60.0,
             capacity: int = 0, epoch_samples: int = 0, spot_price_per_hour: float = 0.0,
             ondemand_price_per_hour: float = 0.0, planner: Optional["Planner"] = None, device: int = 0):
    """run(series, w, policy, seed, options, shared_planner) (simulator.cpp:119-340).
    Returns (report dict, list of per-interval dicts) with the reference's
    report_to_json field names."""
    lib = _abi.lib()
    p, keep = w.to_c()
    c = (costs or CostTable()).to_c()
    o = (opt or PlannerOptions()).to_c()
    n = len(counts)
    cnt = (C.c_int32 * max(n, 1))(*counts)
    rep = _abi.lp_sim_report()
    logs = (_abi.lp_interval_log * max(n, 1))()
    _abi.check(lib.lp_simulate(planner._h if planner else None, C.byref(p), C.byref(c), C.byref(o), device, cnt, n,
                               interval_s, capacity, C.byref(pol), seed, epoch_samples, spot_price_per_hour,
                               ondemand_price_per_hour, C.byref(rep), logs))
    return _report_dicts(rep, logs, n)
