"""Zebra-parallel task DAG: the per-(layer, microbatch) chain the B200 executor walks.

Drop-in for ``zpsim.taskgraph`` (``/root/reference/pkg/src/zpsim/taskgraph.py``). Task ids,
kinds, lanes, durations and edges are identical to the reference for the same inputs (ids
are insertion order, so the construction order below is part of the contract: the forward
sweep layer by layer — all AttnF of the layer, then per microbatch Disp/Exp/Comb[/OffExp] —
then the backward sweep from layer L down).

On B200 each kind maps to real work: ATTN_F = combine(l-1) + attention +
router + dispatch permute; DISP_F / COMB_F = NCCL all-to-all; EXP_F / OFF_EXP_F = grouped
SwiGLU FFN; the backward kinds mirror them.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from fractions import Fraction
from typing import Optional, Sequence

from .core import ExpertAssignment, InfeasibleError, Spec, TaskDurations, ValidationError, round_ns

ATTN_DEVICE = "attn"
EXP_DEVICE = "exp"
COMPUTE = "compute"
DISPATCH = "dispatch"
COMBINE = "combine"


class TaskKind(str, Enum):
    ATTN_F = "AttnF"
    ATTN_B = "AttnB"
    EXP_F = "ExpF"
    EXP_B = "ExpB"
    OFF_EXP_F = "OffExpF"
    OFF_EXP_B = "OffExpB"
    DISP_F = "DispF"
    DISP_B = "DispB"
    COMB_F = "CombF"
    COMB_B = "CombB"


K = TaskKind
COMPUTE_KINDS = {K.ATTN_F, K.ATTN_B, K.EXP_F, K.EXP_B, K.OFF_EXP_F, K.OFF_EXP_B}
OFFLOAD_KINDS = {K.OFF_EXP_F, K.OFF_EXP_B}

# kind -> (device, lane). Dispatch sits on the sending attention device, combine on the
# sending expert device (reference taskgraph.py:49-60).
_KIND_PLACEMENT = {
    **{k: (ATTN_DEVICE, COMPUTE) for k in (K.ATTN_F, K.ATTN_B, K.OFF_EXP_F, K.OFF_EXP_B)},
    **{k: (EXP_DEVICE, COMPUTE) for k in (K.EXP_F, K.EXP_B)},
    K.DISP_F: (ATTN_DEVICE, DISPATCH),
    K.DISP_B: (ATTN_DEVICE, DISPATCH),
    K.COMB_F: (EXP_DEVICE, COMBINE),
    K.COMB_B: (EXP_DEVICE, COMBINE),
}


@dataclass(frozen=True)
class Task:
    id: int
    kind: TaskKind
    layer: int
    microbatch: int
    device: str
    lane: tuple
    duration: int


@dataclass
class TaskGraph:
    """DAG of lane-bound tasks; treat as immutable once built."""

    mode: str
    layers: int
    microbatches: int
    tasks: tuple
    edges: tuple
    assignment: ExpertAssignment
    forward_only: bool = False
    _index: dict = field(default_factory=dict, repr=False)
    _succ: dict = field(default_factory=dict, repr=False)
    _pred: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        self._index = {(t.kind, t.layer, t.microbatch): t.id for t in self.tasks}
        self._succ = {t.id: [] for t in self.tasks}
        self._pred = {t.id: [] for t in self.tasks}
        for u, v in self.edges:
            self._succ[u].append(v)
            self._pred[v].append(u)
        _assert_acyclic(self)

    def task(self, kind: TaskKind, layer: int, microbatch: int) -> Task:
        return self.tasks[self._index[(kind, layer, microbatch)]]

    def has(self, kind: TaskKind, layer: int, microbatch: int) -> bool:
        return (kind, layer, microbatch) in self._index

    def successors(self, task_id: int):
        return self._succ[task_id]

    def predecessors(self, task_id: int):
        return self._pred[task_id]

    def lanes(self):
        return list(dict.fromkeys(t.lane for t in self.tasks))

    def tasks_on(self, lane):
        return [t for t in self.tasks if t.lane == lane]


def _assert_acyclic(graph: TaskGraph) -> None:
    indeg = {t.id: len(graph._pred[t.id]) for t in graph.tasks}
    stack = [i for i in sorted(indeg) if indeg[i] == 0]
    visited = 0
    while stack:
        u = stack.pop()
        visited += 1
        for v in graph._succ[u]:
            indeg[v] -= 1
            if indeg[v] == 0:
                stack.append(v)
    if visited != len(graph.tasks):
        raise ValidationError(["task graph contains a dependency cycle"])


def offload_scaling(spec: Spec, assignment: ExpertAssignment):
    """Per layer: expert-GPU time scale 1 - o*N/n and attention-side share o*N^2/(n*M)."""
    n, M, N = spec.model.experts_per_layer, spec.cluster.attention_gpus, spec.cluster.expert_gpus
    scales, shares = [], []
    for o in assignment.offload:
        if not 0 <= o <= n // N:
            raise ValidationError([f"offload count {o} outside [0, {n // N}]"])
        scales.append(1 - Fraction(o * N, n))
        shares.append(Fraction(o * N * N, n * M))
    return scales, shares


def _check_chunks(spec: Spec, assignment: ExpertAssignment) -> None:
    if not any(assignment.offload):
        return
    from .scheduler import chunk_sizes

    _, n2 = chunk_sizes(spec.cluster.attention_gpus, spec.cluster.expert_gpus)
    bad = [o for o in assignment.offload if o % n2]
    if bad:
        raise ValidationError([f"offload counts {bad} are not multiples of chunk size n_2={n2}"])


class _GraphBuilder:
    def __init__(self):
        self.tasks = []
        self.ids = {}
        self.edges = set()

    def add(self, kind, layer, mb, duration):
        device, lane = _KIND_PLACEMENT[kind]
        tid = len(self.tasks)
        self.tasks.append(Task(tid, kind, layer, mb, device, (device, lane), int(duration)))
        self.ids[(kind, layer, mb)] = tid

    def dep(self, a, b):
        self.edges.add((self.ids[a], self.ids[b]))

    def graph(self, mode, layers, mbs, assignment, forward_only):
        return TaskGraph(mode, layers, mbs, tuple(self.tasks), tuple(sorted(self.edges)),
                         assignment, forward_only)


def build_zp_graph(
    spec: Spec,
    durations: TaskDurations,
    assignment: Optional[ExpertAssignment] = None,
    mode: Optional[str] = None,
    include_backward: bool = True,
) -> TaskGraph:
    """ZP DAG (reference taskgraph.py:209-320).

    Forward per (l, j): AttnF -> DispF -> ExpF -> CombF -> AttnF(l+1); backward mirrors it.
    zp-theorem keeps expert tasks on layers 1..L-1 and turns around at AttnF(L) -> AttnB(L);
    zp-full keeps layer-L experts, with the loss edge CombF(L) -> DispB(L). Offloaded
    experts run on the attention device, gated by the dispatch, joining the combine.
    """
    mode = mode or spec.run.mode
    if mode not in ("zp-theorem", "zp-full"):
        raise ValueError(f"unknown ZP graph mode {mode!r}")
    L, R = spec.model.layers, spec.model.microbatches
    assignment = assignment or ExpertAssignment.zeros(L)
    if len(assignment.offload) != L:
        raise ValidationError([f"assignment has {len(assignment.offload)} entries for {L} layers"])
    if mode == "zp-theorem" and assignment.offload[-1] > 0:
        raise ValidationError(["zp-theorem mode has no layer-" + str(L) + " expert tasks to offload"])
    _check_chunks(spec, assignment)
    scales, shares = offload_scaling(spec, assignment)

    gamma = durations.backward_factor
    t_exp = Fraction(durations.expert_layer_fwd_on_expert_gpu)
    t_single = Fraction(durations.single_expert_fwd_on_attn_gpu)
    last_expert_layer = L - 1 if mode == "zp-theorem" else L

    def per_layer(l):
        """(ExpF, ExpB, OffExpF, OffExpB) durations of layer l."""
        sc, sh = scales[l - 1], shares[l - 1]
        return (round_ns(t_exp * sc), round_ns(gamma * t_exp * sc),
                round_ns(t_single * sh), round_ns(gamma * t_single * sh))

    g = _GraphBuilder()
    mbs = range(1, R + 1)
    for l in range(1, L + 1):
        for j in mbs:
            g.add(K.ATTN_F, l, j, durations.attn_fwd)
            if l > 1:
                g.dep((K.COMB_F, l - 1, j), (K.ATTN_F, l, j))
        if l > last_expert_layer:
            continue
        exp_f, _, off_f, _ = per_layer(l)
        off = assignment.offload[l - 1] > 0
        for j in mbs:
            g.add(K.DISP_F, l, j, durations.dispatch)
            g.add(K.EXP_F, l, j, exp_f)
            g.dep((K.ATTN_F, l, j), (K.DISP_F, l, j))
            g.dep((K.DISP_F, l, j), (K.EXP_F, l, j))
            g.add(K.COMB_F, l, j, durations.combine)
            g.dep((K.EXP_F, l, j), (K.COMB_F, l, j))
            if off:
                g.add(K.OFF_EXP_F, l, j, off_f)
                g.dep((K.DISP_F, l, j), (K.OFF_EXP_F, l, j))
                g.dep((K.OFF_EXP_F, l, j), (K.COMB_F, l, j))
    if include_backward:
        attn_b = round_ns(gamma * durations.attn_fwd)
        disp_b = round_ns(gamma * durations.dispatch)
        comb_b = round_ns(gamma * durations.combine)
        for l in range(L, 0, -1):
            for j in mbs:
                g.add(K.ATTN_B, l, j, attn_b)
            if l > last_expert_layer:
                continue
            _, exp_b, _, off_b = per_layer(l)
            off = assignment.offload[l - 1] > 0
            for j in mbs:
                g.add(K.DISP_B, l, j, disp_b)
                g.add(K.EXP_B, l, j, exp_b)
                g.add(K.COMB_B, l, j, comb_b)
                for a, b in ((K.DISP_B, K.EXP_B), (K.EXP_B, K.COMB_B), (K.COMB_B, K.ATTN_B)):
                    g.dep((a, l, j), (b, l, j))
                if off:
                    g.add(K.OFF_EXP_B, l, j, off_b)
                    g.dep((K.DISP_B, l, j), (K.OFF_EXP_B, l, j))
                    g.dep((K.OFF_EXP_B, l, j), (K.COMB_B, l, j))
                # layer L: the loss turnaround waits for the combined forward output
                src = (K.COMB_F, l, j) if l == L else (K.ATTN_B, l + 1, j)
                g.dep(src, (K.DISP_B, l, j))
        if mode == "zp-theorem":
            for j in mbs:
                g.dep((K.ATTN_F, L, j), (K.ATTN_B, L, j))
    return g.graph(mode, L, R, assignment, not include_backward)


def build_distep_graph(spec: Spec, durations: TaskDurations, include_backward: bool = True) -> TaskGraph:
    """DistEP lockstep ablation: the zp-full graph plus serialisation edges so no device works
    on (l, j+1) before (l, j)'s combine lands (reference taskgraph.py:323-369)."""
    base = build_zp_graph(spec, durations, None, "zp-full", include_backward)
    L, R = base.layers, base.microbatches
    tid = lambda kind, l, j: base.task(kind, l, j).id  # noqa: E731
    edges = set(base.edges)
    for l in range(1, L + 1):
        edges.update((tid(K.COMB_F, l, j), tid(K.ATTN_F, l, j + 1)) for j in range(1, R))
        if l < L:
            edges.add((tid(K.COMB_F, l, R), tid(K.ATTN_F, l + 1, 1)))
    if include_backward:
        edges.add((tid(K.COMB_F, L, R), tid(K.DISP_B, L, 1)))
        for l in range(L, 0, -1):
            edges.update((tid(K.ATTN_B, l, j), tid(K.DISP_B, l, j + 1)) for j in range(1, R))
            if l > 1:
                edges.add((tid(K.ATTN_B, l, R), tid(K.DISP_B, l - 1, 1)))
    return TaskGraph("distep", L, R, base.tasks, tuple(sorted(edges)), base.assignment,
                     not include_backward)


def token_flow(spec: Spec, assignment: ExpertAssignment, layer: int) -> dict:
    """Routed-token split of one (layer, microbatch) and its conservation."""
    from .costmodel import routed_tokens_per_microbatch

    total = Fraction(routed_tokens_per_microbatch(spec))
    share = Fraction(assignment.offload[layer - 1] * spec.cluster.expert_gpus,
                     spec.model.experts_per_layer)
    to_off = total * share
    return {"entering_dispatch": total, "to_expert_gpus": total - to_off,
            "to_offloaded_experts": to_off, "leaving_combine": total}


def graph_to_json(graph: TaskGraph) -> dict:
    return {
        "mode": graph.mode,
        "layers": graph.layers,
        "microbatches": graph.microbatches,
        "forward_only": graph.forward_only,
        "offload": list(graph.assignment.offload),
        "tasks": [{"id": t.id, "kind": t.kind.value, "layer": t.layer, "microbatch": t.microbatch,
                   "device": t.device, "lane": list(t.lane), "duration": t.duration}
                  for t in graph.tasks],
        "edges": [list(e) for e in graph.edges],
    }
