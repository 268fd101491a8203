"""ctypes mirror of include/liveput.h and the loader for libliveput.so.

The product path is the CUDA library built from ``csrc/`` (sm_100a).  There is
no CPU fallback: if the shared library is missing, or a call is made on a box
without a GPU, the call fails loudly (ImportError / LiveputError).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "lib" / "libliveput.so"

LP_OK, LP_EINVAL, LP_ECUDA, LP_ENOMEM, LP_EUNSUPPORTED, LP_ENCCL, LP_EROLLBACK = range(7)
LP_MIG_NONE, LP_MIG_INTRA_STAGE, LP_MIG_INTER_STAGE, LP_MIG_PIPELINE = range(4)
LP_PREDICT_ARIMA, LP_PREDICT_MOVING_AVG, LP_PREDICT_EXP_SMOOTH, LP_PREDICT_LAST_VALUE = range(4)
LP_POLICY_PROACTIVE, LP_POLICY_IDEAL, LP_POLICY_REACTIVE, LP_POLICY_CHECKPOINT, LP_POLICY_REDUNDANCY = range(5)
LP_NCCL_ID_BYTES = 128


class lp_config(C.Structure):
    _fields_ = [("pipelines", C.c_int32), ("stages", C.c_int32)]


class lp_profile(C.Structure):
    _fields_ = [
        ("compute_per_microbatch_s", C.c_double),
        ("param_bytes", C.c_double),
        ("activation_bytes", C.c_double),
        ("minibatch_size", C.c_int32),
        ("microbatch_size", C.c_int32),
        ("device_memory_bytes", C.c_double),
        ("memory_fixed_bytes", C.c_double),
        ("memory_per_stage_bytes", C.c_double),
        ("alpha_s", C.c_double),
        ("beta_s_per_byte", C.c_double),
        ("n_rates", C.c_int32),
        ("rate_depths", C.POINTER(C.c_int32)),
        ("rate_values", C.POINTER(C.c_double)),
    ]


class lp_costs(C.Structure):
    _fields_ = [
        ("start_process_s", C.c_double),
        ("rendezvous_s", C.c_double),
        ("cuda_context_s", C.c_double),
        ("load_data_s", C.c_double),
        ("build_model_s", C.c_double),
        ("update_comm_groups_s", C.c_double),
    ]


class lp_options(C.Structure):
    _fields_ = [
        ("interval_s", C.c_double),
        ("lookahead", C.c_int32),
        ("mc_trials", C.c_int32),
        ("exact_cap", C.c_uint64),
        ("mc_seed", C.c_uint64),
        ("rollback_penalty_s", C.c_double),
        ("strict_conditional", C.c_int32),
    ]


class lp_plan_step(C.Structure):
    _fields_ = [
        ("interval_index", C.c_int32),
        ("config", lp_config),
        ("expected_committed", C.c_double),
        ("expected_mig_cost_s", C.c_double),
    ]


class lp_liveput_row(C.Structure):
    _fields_ = [("interval", C.c_int32), ("config", lp_config), ("liveput", C.c_double)]


class lp_stats(C.Structure):
    _fields_ = [
        ("resolutions", C.c_uint64),
        ("scenarios", C.c_uint64),
        ("local_scenarios", C.c_uint64),
        ("mc_pairs", C.c_int32),
        ("exact_pairs", C.c_int32),
        ("kernel_launches", C.c_int32),
        ("horizon", C.c_int32),
        ("hist_ms", C.c_double),
        ("reduce_ms", C.c_double),
        ("dp_ms", C.c_double),
        ("total_ms", C.c_double),
        ("hist_alg_ops", C.c_uint64),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("prepare_ms", C.c_double),
        ("cached_pairs", C.c_uint64),
        ("hist_survey_ops", C.c_uint64),
    ]


class lp_move(C.Structure):
    _fields_ = [("instance", C.c_int32), ("from_pipeline", C.c_int32), ("from_stage", C.c_int32),
                ("to_pipeline", C.c_int32), ("to_stage", C.c_int32), ("transfers_params", C.c_int32)]


class lp_migration(C.Structure):
    _fields_ = [("kind", C.c_int32), ("transfer_rounds", C.c_int32), ("source", lp_config),
                ("target", lp_config), ("est_cost_s", C.c_double), ("n_moves", C.c_int32),
                ("pad", C.c_int32)]


class lp_forecast_config(C.Structure):
    _fields_ = [("history_len", C.c_int32), ("lookahead", C.c_int32), ("capacity", C.c_int32),
                ("floor", C.c_int32), ("max_step", C.c_int32), ("reset_threshold", C.c_int32),
                ("moving_avg_window", C.c_int32), ("pad", C.c_int32), ("exp_smooth_factor", C.c_double),
                ("steep_decay", C.c_double)]


class lp_policy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lookahead", C.c_int32), ("method", C.c_int32), ("history", C.c_int32),
                ("ckpt_period_intervals", C.c_int32), ("redundancy_fixed_stages", C.c_int32),
                ("ckpt_save_cost_s", C.c_double), ("ckpt_restore_cost_s", C.c_double),
                ("ckpt_restart_cost_s", C.c_double), ("redundancy_slowdown", C.c_double)]


class lp_ledger(C.Structure):
    _fields_ = [("effective_s", C.c_double), ("migration_s", C.c_double), ("checkpoint_s", C.c_double),
                ("wasted_rollback_s", C.c_double), ("idle_s", C.c_double)]


class lp_interval_log(C.Structure):
    _fields_ = [("interval", C.c_int32), ("available", C.c_int32), ("pipelines", C.c_int32),
                ("stages", C.c_int32), ("throughput", C.c_double), ("committed", C.c_int64),
                ("rolled_back", C.c_int64), ("migration", C.c_int32), ("pad", C.c_int32), ("ledger", lp_ledger)]


class lp_sim_report(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("committed_samples", C.c_int64), ("wall_time_s", C.c_double),
                ("ledger", lp_ledger), ("instance_seconds", C.c_double), ("instance_hours", C.c_double),
                ("spot_cost", C.c_double), ("ondemand_cost", C.c_double), ("cost_per_sample", C.c_double),
                ("has_cost_per_sample", C.c_int32), ("epochs_completed", C.c_int32),
                ("rollback_events", C.c_int32), ("suspended_intervals", C.c_int32),
                ("sample_accounting_ok", C.c_int32), ("pad", C.c_int32)]


class LiveputError(RuntimeError):
    pass


class RollbackRequired(LiveputError):
    """migration.hpp:49-51: a stage lost every replica; restore from checkpoint."""


_lib = None

# name -> (restype, argtypes); every symbol include/liveput.h declares.
_P = C.POINTER
_SIGS = {
    "lp_create": (C.c_int, [_P(lp_profile), _P(lp_costs), _P(lp_options), C.c_int32, _P(C.c_void_p)]),
    "lp_destroy": (None, [C.c_void_p]),
    "lp_last_error": (C.c_char_p, [C.c_void_p]),
    "lp_last_global_error": (C.c_char_p, []),
    "lp_get_options": (C.c_int, [C.c_void_p, _P(lp_options)]),
    "lp_replan": (C.c_int, [C.c_void_p, lp_config, _P(C.c_int32), C.c_int32, _P(lp_plan_step),
                            _P(lp_liveput_row), C.c_int32, _P(C.c_int32)]),
    "lp_prepare": (C.c_int, [C.c_void_p, lp_config, _P(C.c_int32), C.c_int32]),
    "lp_execute": (C.c_int, [C.c_void_p]),
    "lp_fetch": (C.c_int, [C.c_void_p, _P(lp_plan_step), _P(lp_liveput_row), C.c_int32, _P(C.c_int32)]),
    "lp_get_stats": (C.c_int, [C.c_void_p, _P(lp_stats)]),
    "lp_stream": (C.c_void_p, [C.c_void_p]),
    "lp_set_hist_cache": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64]),
    "lp_precompute": (C.c_int, [C.c_void_p, _P(C.c_int32), _P(C.c_int32), C.c_int32]),
    "lp_cache_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, _P(C.c_uint64)]),
    "lp_cache_import": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "lp_phi": (C.c_int, [C.c_void_p, lp_config, lp_config, C.c_int32, C.c_int32, _P(C.c_double), _P(C.c_double)]),
    "lp_sequence_value": (C.c_int, [C.c_void_p, lp_config, _P(lp_config), _P(C.c_int32), C.c_int32, _P(C.c_double)]),
    "lp_survivor_hist": (C.c_int, [C.c_void_p, lp_config, C.c_int32, C.c_int32, _P(C.c_uint64), _P(C.c_uint64)]),
    "lp_expected_liveput": (C.c_int, [C.c_void_p, lp_config, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64, _P(C.c_double)]),
    "lp_dump_survivors": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64,
                                    _P(lp_config), C.c_int32, _P(C.c_uint16)]),
    "lp_dump_scenarios": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_uint64, _P(C.c_uint16)]),
    "lp_nccl_unique_id": (C.c_int, [_P(C.c_uint8)]),
    "lp_comm_init": (C.c_int, [C.c_void_p, _P(C.c_uint8), C.c_int32, C.c_int32]),
    "lp_set_shard": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    "lp_throughput": (C.c_double, [_P(lp_profile), lp_config]),
    "lp_depth_feasible": (C.c_int32, [_P(lp_profile), C.c_int32]),
    "lp_enumerate_configs": (C.c_int32, [_P(lp_profile), C.c_int32, _P(lp_config), C.c_int32]),
    "lp_reactive_plan": (C.c_int32, [_P(lp_profile), C.c_int32, _P(lp_config)]),
    "lp_scenario_count": (C.c_uint64, [C.c_int32, C.c_int32]),
    "lp_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "lp_plan_migration": (C.c_int, [_P(lp_profile), _P(lp_costs), lp_config, C.c_int32, _P(C.c_uint8),
                                    C.c_int32, lp_config, _P(lp_migration), _P(lp_move), C.c_int32]),
    "lp_migration_cost": (C.c_double, [_P(lp_profile), _P(lp_costs), _P(lp_migration), C.c_int32]),
    "lp_transition_outcome": (C.c_int, [_P(lp_profile), _P(lp_costs), C.c_int32, lp_config, lp_config,
                                        C.c_int32, _P(C.c_double), _P(C.c_int32), _P(C.c_int32)]),
    "lp_resume_cost": (C.c_double, [_P(lp_profile), _P(lp_costs), lp_config]),
    "lp_forecast_defaults": (lp_forecast_config, [C.c_int32]),
    "lp_predict": (C.c_int, [_P(C.c_int32), C.c_int32, _P(lp_forecast_config), C.c_int32, C.c_int32,
                             _P(C.c_int32)]),
    "lp_predict_windows": (C.c_int, [_P(C.c_int32), C.c_int32, _P(lp_forecast_config), _P(C.c_int32), C.c_int32,
                                     C.c_int32, _P(C.c_int32), _P(C.c_double), _P(C.c_int32)]),
    "lp_eval_l1": (C.c_double, [_P(C.c_int32), _P(C.c_int32), C.c_int32]),
    "lp_policy_defaults": (lp_policy, [C.c_int32]),
    "lp_simulate": (C.c_int, [C.c_void_p, _P(lp_profile), _P(lp_costs), _P(lp_options), C.c_int32, _P(C.c_int32),
                              C.c_int32, C.c_double, C.c_int32, _P(lp_policy), C.c_uint64, C.c_int32, C.c_double,
                              C.c_double, _P(lp_sim_report), _P(lp_interval_log)]),
    "lp_simulate_batch": (C.c_int, [C.c_void_p, _P(lp_profile), _P(lp_costs), _P(lp_options), C.c_int32,
                                    _P(C.c_int32), C.c_int32, C.c_double, C.c_int32, _P(lp_policy), _P(C.c_uint64),
                                    C.c_int32, C.c_int32, C.c_double, C.c_double, _P(lp_sim_report),
                                    _P(lp_interval_log)]),
    "lp_max_instances": (C.c_int32, []),
    "lp_build_info": (C.c_char_p, []),
}


def exported_symbols():
    return list(_SIGS)


def lib():
    """Load libliveput.so (in-tree build).  Raises ImportError if it is missing:
    the product path has no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("LIVEPUT_LIB", LIB_PATH))
    if not path.exists():
        raise ImportError(
            f"liveput CUDA library not built: {path} is missing. "
            "Run `python -c 'import __graft_entry__ as g; g.build()'` or `make -C paper_2403_14097_b200/csrc`."
        )
    if not os.environ.get("LIVEPUT_NCCL_LIB"):
        # bind the same NCCL torch uses (the library dlopens it lazily)
        try:
            import importlib.util
            spec = importlib.util.find_spec("nvidia.nccl")
            if spec and spec.submodule_search_locations:
                cand = Path(list(spec.submodule_search_locations)[0]) / "lib" / "libnccl.so.2"
                if cand.exists():
                    os.environ["LIVEPUT_NCCL_LIB"] = str(cand)
        except Exception:
            pass
    l = C.CDLL(str(path))
    for name, (res, args) in _SIGS.items():
        fn = getattr(l, name)
        fn.restype = res
        fn.argtypes = args
    _lib = l
    return l


def check(status, handle=None):
    if status == LP_OK:
        return
    l = lib()
    msg = l.lp_last_error(handle) if handle else l.lp_last_global_error()
    msg = msg.decode() if msg else ""
    if status == LP_EINVAL:
        raise ValueError(msg)
    if status == LP_EROLLBACK:
        raise RollbackRequired(msg)
    raise LiveputError(f"liveput status {status}: {msg}")
