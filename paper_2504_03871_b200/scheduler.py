"""Zebra stream orders and the Asym-EA "gather and squeeze" offload planner.

Drop-in for the hot-path half of ``zpsim.scheduler``
(``/root/reference/pkg/src/zpsim/scheduler.py:26-312``): ``chunk_sizes``, the Theorem
compute-lane order ``zp_compute_order``, ``comm_order``, ``default_orders`` (+ the DistEP
lockstep orders), and Algorithm 1 ``asym_ea_offload`` in exact rationals. The brute-force
search oracles of the reference are test infrastructure and are not re-implemented; the
parity tests compare against the reference's own outputs (``tests/golden``).

``default_orders(graph)`` is exactly what the B200 executor (``executor.py``) walks: each
rank issues its role's lanes in this order, so collectives are posted in the same order on
every rank.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from typing import Optional

from .core import ExpertAssignment, InfeasibleError, ValidationError, as_fraction
from .taskgraph import ATTN_DEVICE, COMBINE, COMPUTE, DISPATCH, EXP_DEVICE, TaskGraph, TaskKind

K = TaskKind
ATTN_LANE = (ATTN_DEVICE, COMPUTE)
EXP_LANE = (EXP_DEVICE, COMPUTE)
DISP_LANE = (ATTN_DEVICE, DISPATCH)
COMB_LANE = (EXP_DEVICE, COMBINE)


def chunk_sizes(attention_gpus: int, expert_gpus: int):
    """(n_1, n_2): experts acquired per attention GPU / given up per expert GPU per chunk.
    Needs M | N or N | M (reference scheduler.py:36-44)."""
    M, N = attention_gpus, expert_gpus
    if M < 1 or N < 1 or (M % N and N % M):
        raise ValidationError([f"chunk sizes need M % N == 0 or N % M == 0, got M={M}, N={N}"])
    n1 = max(1, N // M)
    return n1, n1 * M // N


# ---------------------------------------------------------------------------------------------
# stream orders


def zp_compute_order(graph: TaskGraph) -> dict:
    """Theorem schedule for the two compute lanes (reference scheduler.py:51-107).

    Attention lane: forward layers 1..L-1 microbatch-major (offloaded experts after each
    layer's block), the layer-L forward/backward turnaround interleaved per microbatch, then
    backward layers L-1..1 (offloaded experts before each block). Expert lane: forward layers
    ascending, layer L fwd/bwd interleaved (zp-full), backward layers descending.
    """
    if graph.mode not in ("zp-theorem", "zp-full"):
        raise ValueError(f"zp_compute_order needs a ZP graph, got mode {graph.mode!r}")
    L, R = graph.layers, graph.microbatches
    bwd = not graph.forward_only
    mbs = range(1, R + 1)

    def ids(kind, l):
        return [graph.task(kind, l, j).id for j in mbs if graph.has(kind, l, j)]

    attn = []
    for l in range(1, L):
        attn += ids(K.ATTN_F, l) + ids(K.OFF_EXP_F, l)
    if bwd:
        for j in mbs:
            for kind in (K.ATTN_F, K.OFF_EXP_F, K.OFF_EXP_B, K.ATTN_B):
                if graph.has(kind, L, j):
                    attn.append(graph.task(kind, L, j).id)
        for l in range(L - 1, 0, -1):
            attn += ids(K.OFF_EXP_B, l) + ids(K.ATTN_B, l)
    else:
        attn += ids(K.ATTN_F, L) + ids(K.OFF_EXP_F, L)

    exp = []
    for l in range(1, L):
        exp += ids(K.EXP_F, l)
    if graph.has(K.EXP_F, L, 1):
        for j in mbs:
            exp.append(graph.task(K.EXP_F, L, j).id)
            if bwd:
                exp.append(graph.task(K.EXP_B, L, j).id)
    if bwd:
        for l in range(L - 1, 0, -1):
            exp += ids(K.EXP_B, l)
    return {ATTN_LANE: attn, EXP_LANE: exp}


def comm_order(graph: TaskGraph, compute_order: dict) -> dict:
    """Each transfer follows its producer's compute-lane position; key (pos, fwd0/bwd1, id)
    (reference scheduler.py:110-140)."""
    apos = {tid: i for i, tid in enumerate(compute_order.get(ATTN_LANE, []))}
    epos = {tid: i for i, tid in enumerate(compute_order.get(EXP_LANE, []))}
    L = graph.layers
    disp, comb = [], []
    for t in graph.tasks:
        l, j = t.layer, t.microbatch
        if t.kind is K.DISP_F:
            disp.append((apos[graph.task(K.ATTN_F, l, j).id], 0, t.id))
        elif t.kind is K.DISP_B:
            prod = graph.task(K.ATTN_B, l + 1, j) if l < L else graph.task(K.ATTN_F, L, j)
            disp.append((apos[prod.id], 1, t.id))
        elif t.kind is K.COMB_F:
            comb.append((epos[graph.task(K.EXP_F, l, j).id], 0, t.id))
        elif t.kind is K.COMB_B:
            comb.append((epos[graph.task(K.EXP_B, l, j).id], 0, t.id))
    return {DISP_LANE: [k[2] for k in sorted(disp)], COMB_LANE: [k[2] for k in sorted(comb)]}


def distep_orders(graph: TaskGraph) -> dict:
    """Lockstep orders: layer- then microbatch-serial (reference scheduler.py:143-160)."""
    L, R = graph.layers, graph.microbatches
    bwd = not graph.forward_only

    def sweep(kind, layers):
        return [graph.task(kind, l, j).id for l in layers for j in range(1, R + 1)]

    fwd_l, bwd_l = range(1, L + 1), range(L, 0, -1)
    out = {}
    for lane, (kf, kb) in ((ATTN_LANE, (K.ATTN_F, K.ATTN_B)), (EXP_LANE, (K.EXP_F, K.EXP_B)),
                           (DISP_LANE, (K.DISP_F, K.DISP_B)), (COMB_LANE, (K.COMB_F, K.COMB_B))):
        out[lane] = sweep(kf, fwd_l) + (sweep(kb, bwd_l) if bwd else [])
    return out


def default_orders(graph: TaskGraph) -> dict:
    """Complete StreamOrder: compute lanes plus comm lanes."""
    if graph.mode == "distep":
        return distep_orders(graph)
    orders = zp_compute_order(graph)
    orders.update(comm_order(graph, orders))
    return orders


# ---------------------------------------------------------------------------------------------
# Asym-EA (Algorithm 1, "gather and squeeze")


@dataclass(frozen=True)
class OffloadPlanInputs:
    experts_per_layer: int
    layers: int
    attention_gpus: int
    expert_gpus: int
    attn_fwd: Fraction
    single_expert_on_attn: Fraction
    expert_layer_on_expert: Fraction
    n_min: int = 0
    n_max: Optional[int] = None
    squeeze_mode: str = "verbatim"


@dataclass(frozen=True)
class OffloadPlan:
    assignment: ExpertAssignment
    chunk: tuple
    t_gather: Fraction
    t_squeeze: Fraction
    alpha: Fraction
    beta: Fraction
    residuals: tuple
    note: str = ""


def asym_ea_offload(inputs: OffloadPlanInputs) -> OffloadPlan:
    """Gather the per-layer bubble T_gather = T_exp - T_attn; whenever the ledger holds at
    least one chunk's worth T_squeeze, offload floor(ledger / T_squeeze) chunks at that layer.
    Memory bounds scale the gather rate by alpha (n_max) or beta (n_min). Exact rationals
    (reference scheduler.py:205-293)."""
    n, L = inputs.experts_per_layer, inputs.layers
    if n < 1 or L < 1:
        raise ValidationError(["offload inputs need n >= 1 and L >= 1"])
    n1, n2 = chunk_sizes(inputs.attention_gpus, inputs.expert_gpus)
    t_attn, t_single, t_exp = (as_fraction(v) for v in
                               (inputs.attn_fwd, inputs.single_expert_on_attn, inputs.expert_layer_on_expert))
    if min(t_attn, t_single, t_exp) < 0:
        raise ValidationError(["offload input times must be >= 0"])
    if inputs.squeeze_mode not in ("verbatim", "rederived"):
        raise ValueError(f"unknown squeeze mode {inputs.squeeze_mode!r}")

    N = inputs.expert_gpus
    on_exp = t_exp * N / n  # one expert's tokens on an expert GPU
    on_attn = t_single * N / n  # one acquired expert on an attention GPU
    f_exp, f_attn = (n1, n2) if inputs.squeeze_mode == "verbatim" else (n2, n1)
    t_squeeze = on_exp * f_exp + on_attn * f_attn
    t_gather = t_exp - t_attn

    n_min, n_max = max(0, inputs.n_min), inputs.n_max
    need_chunks = math.ceil(Fraction(n_min, n2))
    if n_max is not None:
        if n_min > n_max:
            raise InfeasibleError(f"memory bounds contradict: n_min={n_min} > n_max={n_max}")
        if need_chunks > n_max // n2:
            raise InfeasibleError(
                f"memory bounds admit no whole number of chunks: need ceil({n_min}/{n2}) "
                f"chunks but only floor({n_max}/{n2}) fit")

    if t_gather <= 0:
        if n_min > 0:
            raise InfeasibleError(
                "memory requires offloading but expert GPUs produce no bubbles to gather "
                f"(T_gather={t_gather} <= 0, n_min={n_min})")
        return OffloadPlan(ExpertAssignment.zeros(L), (n1, n2), t_gather, t_squeeze, Fraction(1),
                           Fraction(1), (Fraction(0),) * L, "no bubbles to squeeze")

    budget = L * t_gather
    alpha = Fraction(1) if n_max is None else min(Fraction(n_max // n2) * t_squeeze / budget, Fraction(1))
    beta = max(Fraction(need_chunks) * t_squeeze / budget, Fraction(1))
    if alpha < 1 and beta > 1:
        raise InfeasibleError("alpha and beta both activated: memory bounds are inconsistent")

    rate = alpha * beta * t_gather
    ledger = Fraction(0)
    plan, residuals = [], []
    for _ in range(L):
        ledger += rate
        chunks = ledger // t_squeeze if ledger >= t_squeeze else 0
        ledger -= chunks * t_squeeze
        plan.append(int(chunks) * n2)
        residuals.append(ledger)
    return OffloadPlan(ExpertAssignment(tuple(plan)), (n1, n2), t_gather, t_squeeze, alpha, beta,
                       tuple(residuals))


def compute_l_busy(expert_layer_on_expert, attn_fwd):
    """Layers an expert GPU can lag before attention stalls: T_exp / (T_exp - T_attn)."""
    t_exp, t_attn = as_fraction(expert_layer_on_expert), as_fraction(attn_fwd)
    return math.inf if t_exp <= t_attn else t_exp / (t_exp - t_attn)


def bubble_ledger(inputs: OffloadPlanInputs, layers: Optional[int] = None):
    """Accumulated bubble l * T_gather after each layer without offloading."""
    step = max(as_fraction(inputs.expert_layer_on_expert) - as_fraction(inputs.attn_fwd), Fraction(0))
    return tuple(step * l for l in range(1, (layers if layers is not None else inputs.layers) + 1))
