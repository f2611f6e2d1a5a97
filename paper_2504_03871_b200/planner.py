"""Planner glue on the hot path: tokens/iteration, Algorithm-1 inputs, build+order+simulate.

Drop-in for ``zpsim.planner`` lines 45-87 (``/root/reference/pkg/src/zpsim/planner.py``).
The strategy comparison / sweep machinery of the reference is out of scope.
"""

from __future__ import annotations

from fractions import Fraction
from typing import Optional

from . import costmodel, scheduler, simulator, taskgraph
from .core import ExpertAssignment, Spec, TaskDurations


def tokens_per_iteration(spec: Spec) -> int:
    """Tokens (not top-k copies) per training iteration: s * seqs * M * R."""
    md = spec.model
    return md.seq_len * md.sequences_per_microbatch * spec.cluster.attention_gpus * md.microbatches


def offload_inputs(spec: Spec, durations: TaskDurations,
                   bounds: Optional[costmodel.MemoryBounds] = None) -> scheduler.OffloadPlanInputs:
    b = bounds if bounds is not None else costmodel.memory_bounds(spec)
    return scheduler.OffloadPlanInputs(
        experts_per_layer=spec.model.experts_per_layer,
        layers=spec.model.layers,
        attention_gpus=spec.cluster.attention_gpus,
        expert_gpus=spec.cluster.expert_gpus,
        attn_fwd=Fraction(durations.attn_fwd),
        single_expert_on_attn=Fraction(durations.single_expert_fwd_on_attn_gpu),
        expert_layer_on_expert=Fraction(durations.expert_layer_fwd_on_expert_gpu),
        n_min=b.n_min,
        n_max=b.n_max,
        squeeze_mode=spec.run.squeeze,
    )


def simulate_zp(spec: Spec, durations: TaskDurations, assignment: Optional[ExpertAssignment] = None,
                mode: Optional[str] = None, include_backward: bool = True):
    """Build, order and simulate one ZP instance; returns (graph, timeline)."""
    graph = taskgraph.build_zp_graph(spec, durations, assignment=assignment, mode=mode,
                                     include_backward=include_backward)
    timeline = simulator.simulate(graph, scheduler.default_orders(graph))
    problems = simulator.validate_timeline(graph, timeline)
    if problems:
        raise RuntimeError(f"simulated timeline invalid: {problems}")
    return graph, timeline


def plan_assignment(spec: Spec, durations: TaskDurations) -> ExpertAssignment:
    """Explicit plan > Asym-EA (if enabled) > no offload (the reference CLI's resolution,
    cli.py:93-106)."""
    if spec.run.offload is not None:
        return ExpertAssignment(spec.run.offload)
    if spec.run.asym_ea:
        return scheduler.asym_ea_offload(offload_inputs(spec, durations)).assignment
    return ExpertAssignment.zeros(spec.model.layers)


def clamp_to_layer_capacity(assignment: ExpertAssignment, experts: int, M: int, N: int):
    """Algorithm 1 (``scheduler.asym_ea_offload``, reference ``scheduler.py:264-283``) bounds the
    offload summed over layers (alpha / n_max) but not per layer: with a large bubble (e.g. 3
    attention + 1 expert GPU) it can ask one layer for more experts than an expert GPU holds, which
    ``build_zp_graph`` then rejects (offload outside [0, n/N], reference ``taskgraph.py:178-194``).
    This clamps each layer to the largest whole number of n_2-chunks that fits in n/N and returns
    (assignment, layers clamped). The planner's parity path does not call it; the B200 bench does."""
    _, n2 = scheduler.chunk_sizes(M, N)
    cap = (experts // N) // n2 * n2
    out = tuple(min(o, cap) for o in assignment.offload)
    return ExpertAssignment(out), sum(1 for a, b in zip(assignment.offload, out) if a != b)


def make_zp_spec(M: int, N: int, layers: int, microbatches: int, experts: int, top_k: int,
                 tokens_per_mb: int, hidden: int, attn_fwd_ns: int, expert_layer_fwd_ns: int,
                 single_expert_fwd_ns: int, dispatch_ns: int = 0, combine_ns: int = 0,
                 gamma=Fraction(2), asym_ea: bool = False, squeeze: str = "verbatim",
                 expert_mem: int = 0, attn_capacity: int = 10**12, exp_capacity: int = 10**12,
                 non_expert_mem_attention: int = 0, non_expert_mem_expert: int = 0) -> Spec:
    """Spec with a duration table (measured B200 times enter here, costmodel.py:88-104) and,
    optionally, the measured memory model (``profiler.memory_spec_fields``) that
    ``costmodel.memory_bounds`` turns into the offload bounds n_min / n_max."""
    from .core import GpuClass, HardwareProfile, ModelSpec, RunOptions, ZpGroupSpec

    a = GpuClass("b200-attention", attn_capacity)
    e = GpuClass("b200-expert", exp_capacity)
    prof = HardwareProfile(a, e, {"attn_fwd": int(attn_fwd_ns), "single_expert_fwd": int(single_expert_fwd_ns)},
                           {"expert_layer_fwd": int(expert_layer_fwd_ns)},
                           {"dispatch": int(dispatch_ns), "combine": int(combine_ns)},
                           int(non_expert_mem_attention), int(non_expert_mem_expert))
    model = ModelSpec(layers, experts, top_k, hidden, tokens_per_mb, microbatches, 1, expert_mem, 0)
    return Spec(ZpGroupSpec(M, N, a, e, 900 * 10**9, 2 * hidden), model, prof,
                RunOptions(mode="zp-full", gamma=Fraction(gamma), asym_ea=asym_ea, squeeze=squeeze))
