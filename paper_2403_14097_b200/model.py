"""Host-side planning inputs, mirroring the reference's value types.

WorkloadProfile  perf_model.hpp:26-49     CostTable      migration.hpp:16-27
ParallelConfig   perf_model.hpp:10-16     PlannerOptions optimizer.hpp:13-23
PlanStep         optimizer.hpp:26-31

The three named profiles restate the reference's data files
(proj/data/profiles/{lm_1p5b,lm_6p7b,toy_six_instance}.json, equal to the test
fixtures gpt2ish_profile / gpt3ish_profile / fig_oracle_profile,
tests/support/fixtures.hpp:22-68) and proj/data/costs/default.json, so that
nothing reads /root/reference at run time.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, Optional

from . import _abi


@dataclass(frozen=True)
class ParallelConfig:
    pipelines: int = 1  # D
    stages: int = 1  # P

    def instances(self) -> int:
        return self.pipelines * self.stages

    def to_c(self) -> _abi.lp_config:
        return _abi.lp_config(self.pipelines, self.stages)


def cfg_to_c(cfg: Optional[ParallelConfig]) -> _abi.lp_config:
    """None is the suspended state (the reference's std::nullopt)."""
    return _abi.lp_config(0, 0) if cfg is None else cfg.to_c()


def cfg_from_c(c: _abi.lp_config) -> Optional[ParallelConfig]:
    return None if c.pipelines <= 0 else ParallelConfig(int(c.pipelines), int(c.stages))


@dataclass
class WorkloadProfile:
    name: str = ""
    compute_per_microbatch_s: float = 0.0
    param_bytes: float = 0.0
    activation_bytes: float = 0.0
    minibatch_size: int = 1
    microbatch_size: int = 1
    device_memory_bytes: float = 0.0
    memory_fixed_bytes: float = 0.0
    memory_per_stage_bytes: float = 0.0
    alpha_s: float = 0.0
    beta_s_per_byte: float = 0.0
    pipeline_rates: Dict[int, float] = field(default_factory=dict)

    def to_c(self):
        """Returns (lp_profile, keepalive) — keep the second item alive while the
        struct is in use (it owns the rate arrays)."""
        n = len(self.pipeline_rates)
        depths = (C.c_int32 * max(n, 1))(*sorted(self.pipeline_rates))
        vals = (C.c_double * max(n, 1))(*[self.pipeline_rates[d] for d in sorted(self.pipeline_rates)])
        p = _abi.lp_profile(
            self.compute_per_microbatch_s, self.param_bytes, self.activation_bytes,
            self.minibatch_size, self.microbatch_size, self.device_memory_bytes,
            self.memory_fixed_bytes, self.memory_per_stage_bytes, self.alpha_s,
            self.beta_s_per_byte, n, depths, vals)
        return p, (depths, vals)


@dataclass
class CostTable:
    start_process_s: float = 1.0
    rendezvous_s: float = 5.0
    cuda_context_s: float = 5.0
    load_data_s: float = 5.0
    build_model_s: float = 5.0
    update_comm_groups_s: float = 10.0

    def to_c(self) -> _abi.lp_costs:
        return _abi.lp_costs(self.start_process_s, self.rendezvous_s, self.cuda_context_s,
                             self.load_data_s, self.build_model_s, self.update_comm_groups_s)


@dataclass
class PlannerOptions:
    interval_s: float = 60.0
    lookahead: int = 12
    mc_trials: int = 200
    exact_cap: int = 2000
    mc_seed: int = 0x5EED
    rollback_penalty_s: float = 30.0
    strict_conditional: bool = False

    def to_c(self) -> _abi.lp_options:
        return _abi.lp_options(self.interval_s, self.lookahead, self.mc_trials, self.exact_cap,
                               self.mc_seed, self.rollback_penalty_s, int(self.strict_conditional))


@dataclass
class PlanStep:
    interval_index: int
    config: Optional[ParallelConfig]
    expected_committed: float
    expected_mig_cost_s: float


def lm_1p5b() -> WorkloadProfile:
    """GPT-2 1.5B profile (data/profiles/lm_1p5b.json == gpt2ish_profile); P >= 7."""
    return WorkloadProfile("lm-1.5b", 1.0, 3.0e9, 4.0e7, 128, 1, 16.0e9, 1.5e9, 88.0e9, 5e-3, 2.5e-9)


def lm_6p7b() -> WorkloadProfile:
    """GPT-3 6.7B profile (data/profiles/lm_6p7b.json == gpt3ish_profile); P >= 20."""
    return WorkloadProfile("lm-6.7b", 4.0, 13.4e9, 4.0e7, 64, 1, 16.0e9, 1.0e9, 290.0e9, 5e-3, 2.5e-9)


def toy_six_instance() -> WorkloadProfile:
    """Six-instance rate table (data/profiles/toy_six_instance.json == fig_oracle_profile)."""
    return WorkloadProfile("toy-rate-table", 1.0, 0.0, 0.0, 6, 1, 1.0, 0.0, 2.0, 0.0, 0.0,
                           {2: 30.0, 3: 50.0})


def resnet152_dp() -> WorkloadProfile:
    """Synthesised ResNet-152 data-parallel profile for BASELINE config 2 (the
    reference ships none): 60.2M fp16 parameters, fits at P=1."""
    return WorkloadProfile("resnet152", 0.25, 1.2e8, 0.0, 256, 8, 16.0e9, 4.0e9, 2.0e9, 5e-3, 2.5e-9)


def default_costs() -> CostTable:
    """data/costs/default.json (== CostTable defaults, migration.hpp:16-23)."""
    return CostTable()


PROFILES = {"lm_1p5b": lm_1p5b, "lm_6p7b": lm_6p7b, "toy_six_instance": toy_six_instance,
            "resnet152": resnet152_dp}
