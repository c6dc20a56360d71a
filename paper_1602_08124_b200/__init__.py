"""B200-native vDNN (arXiv 1602.08124): bit-exact planner + CUDA executor.

Python mirror of the reference's network-definition and offload-policy API
(vdnnsim). See include/vdnn.h for the C ABI and DESIGN.md for the design.
"""
from ._lib import VdnnError
from .api import (
    KUNLIMITED_BYTES, AlgoId, AlgoMode, ConfigError, CostModel, DynamicSelection, EventKind, FootprintReport,
    GradientScheme, InvalidDecision, InvalidDepth, JoinRule, LayerKind, NetworkGraph, OomInfo, Phase,
    PolicyDecision, PolicyKind, PoolUseError, ProfilePassResult, RunReport, ShapeMismatch, SimOptions, Stream,
    StreamEvent, TensorShape, UnknownPreset, Violation, WrongLayerKind, baseline_footprint, build_preset,
    dynamic_select, extend_vgg, gradient_map_bytes, greedy_downgrade, per_layer_event_peaks, placements, program_check, replay_check,
    Session, from_bf16_bits, kernel_launch_count, to_bf16_bits, report_from_events, simulate, simulate_oracle, simulate_with_trace, static_decision,
)

__all__ = [n for n in dir() if not n.startswith("_")]
