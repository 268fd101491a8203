"""B200-native liveput planner (Parcae, arxiv 2403.14097): the reference's
``spotsim::Planner`` hot path rebuilt as sm_100a CUDA behind a C ABI
(include/liveput.h).  See DESIGN.md.
"""
from .model import (CostTable, ParallelConfig, PlannerOptions, PlanStep, WorkloadProfile,
                     default_costs, lm_1p5b, lm_6p7b, resnet152_dp, toy_six_instance)

__all__ = ["CostTable", "ParallelConfig", "PlannerOptions", "PlanStep", "WorkloadProfile",
           "default_costs", "lm_1p5b", "lm_6p7b", "resnet152_dp", "toy_six_instance"]


def Planner(*args, **kwargs):  # noqa: N802 — mirrors the reference class name
    from .planner import Planner as _P
    return _P(*args, **kwargs)
