"""B200-native (sm_100a) NRRS per-bounce RRS stage (arXiv 2510.07868).

RRSNet inference on every live path vertex -> normalized RRS factors ->
Mix-Depth gate -> terminate/continue/split decisions written into preallocated
wavefront queues, behind the C ABI in include/nrrs_gpu.h.
"""
from .rrs import (RateControl, SpawnPlan, Strategy, StrategyKind, assignment_name, bernstein_bound,
                  normalize_factors, parse_assignment, parse_strategy, plan_spawns, queue_capacity_for,
                  realize_counts, strategy_name, throughput_rr_factor, uniform_assignment)
from .networks import HashGridSpec, NeuralRrs, NeuralRrsConfig, RrsVariant
from .stage import GpuContext, RrsStage, StageOutputs, StageResult, default_context, strategy_for_depth

__all__ = [
    "RateControl", "SpawnPlan", "Strategy", "StrategyKind", "assignment_name", "bernstein_bound",
    "normalize_factors", "parse_assignment", "parse_strategy", "plan_spawns", "queue_capacity_for",
    "realize_counts", "strategy_name", "throughput_rr_factor", "uniform_assignment", "HashGridSpec",
    "NeuralRrs", "NeuralRrsConfig", "RrsVariant", "GpuContext", "RrsStage", "StageOutputs", "StageResult",
    "default_context", "strategy_for_depth",
]
