"""Known answers of the reference's own test-suite, restated against this package.

Each test cites the reference test it pins (``/root/reference/pkg/tests/...``).
"""

import math
from fractions import Fraction

import pytest

from paper_2504_03871_b200 import (
    DeadlockError,
    ExpertAssignment,
    GpuClass,
    HardwareProfile,
    InfeasibleError,
    ModelSpec,
    OffloadPlanInputs,
    RunOptions,
    Spec,
    TaskDurations,
    TaskKind,
    Timeline,
    ValidationError,
    ZpGroupSpec,
    asym_ea_offload,
    bubble_intervals,
    bubble_ledger,
    build_distep_graph,
    build_zp_graph,
    chunk_sizes,
    comm_order,
    compute_l_busy,
    compute_metrics,
    default_orders,
    derive_task_durations,
    memory_bounds,
    simulate,
    steady_state_utilization,
    token_flow,
    validate_timeline,
    workload_shape,
    zp_compute_order,
)
from paper_2504_03871_b200.scheduler import ATTN_LANE, COMB_LANE, DISP_LANE, EXP_LANE


def spec(M=1, N=1, L=3, R=3, n=6, k=2, attn=3, exp=4, single=3, disp=0, comb=0, gamma=Fraction(1),
         expert_mem=0, attn_cap=10**12, exp_cap=10**12, seq_len=16):
    a, e = GpuClass("fast", attn_cap), GpuClass("slow", exp_cap)
    prof = HardwareProfile(a, e, {"attn_fwd": attn, "single_expert_fwd": single},
                           {"expert_layer_fwd": exp}, {"dispatch": disp, "combine": comb})
    model = ModelSpec(L, n, min(k, n), 64, seq_len, R, 1, expert_mem, 0)
    return Spec(ZpGroupSpec(M, N, a, e, 10**11, 4096), model, prof, RunOptions(gamma=gamma))


def dur(attn=3, exp=4, single=3, disp=0, comb=0, gamma=Fraction(1)):
    return TaskDurations(attn, exp, single, disp, comb, gamma)


def names(g, ids):
    return [f"{g.tasks[t].kind.value}{g.tasks[t].layer},{g.tasks[t].microbatch}" for t in ids]


def fwd(s, d):
    return build_zp_graph(s, d, mode="zp-full", include_backward=False)


# test_scheduler.py:38-51
def test_chunk_sizes():
    assert chunk_sizes(1, 1) == (1, 1) and chunk_sizes(4, 4) == (1, 1)
    assert chunk_sizes(4, 8) == (2, 1)
    assert chunk_sizes(4, 2) == (1, 2)
    with pytest.raises(ValidationError):
        chunk_sizes(4, 3)


# test_scheduler.py:55-85
def test_theorem_lane_orders():
    g = build_zp_graph(spec(L=2, R=2), dur(), mode="zp-theorem")
    o = zp_compute_order(g)
    assert names(g, o[ATTN_LANE]) == ["AttnF1,1", "AttnF1,2", "AttnF2,1", "AttnB2,1", "AttnF2,2",
                                      "AttnB2,2", "AttnB1,1", "AttnB1,2"]
    assert names(g, o[EXP_LANE]) == ["ExpF1,1", "ExpF1,2", "ExpB1,1", "ExpB1,2"]
    g1 = build_zp_graph(spec(L=1, R=3, n=1, k=1), dur(), mode="zp-theorem")
    o1 = zp_compute_order(g1)
    assert names(g1, o1[ATTN_LANE]) == ["AttnF1,1", "AttnB1,1", "AttnF1,2", "AttnB1,2", "AttnF1,3", "AttnB1,3"]
    assert o1[EXP_LANE] == []


# test_scheduler.py:87-102
def test_offload_placement_in_lane():
    g = build_zp_graph(spec(), dur(), assignment=ExpertAssignment((0, 2, 0)), mode="zp-full")
    lane = names(g, zp_compute_order(g)[ATTN_LANE])
    i = lane.index("OffExpF2,1")
    assert lane[i - 1] == "AttnF2,3" and lane[i + 1:i + 3] == ["OffExpF2,2", "OffExpF2,3"]
    g = build_zp_graph(spec(), dur(), assignment=ExpertAssignment((2, 0, 0)), mode="zp-full")
    lane = names(g, zp_compute_order(g)[ATTN_LANE])
    i = lane.index("OffExpB1,1")
    assert lane[i + 3:i + 6] == ["AttnB1,1", "AttnB1,2", "AttnB1,3"]


# test_scheduler.py:106-122
def test_comm_orders():
    g = build_zp_graph(spec(L=2, R=1), dur(), include_backward=False)
    o = comm_order(g, zp_compute_order(g))
    assert names(g, o[DISP_LANE]) == ["DispF1,1", "DispF2,1"]
    assert names(g, o[COMB_LANE]) == ["CombF1,1", "CombF2,1"]
    g = build_zp_graph(spec(L=2, R=2), dur(), mode="zp-theorem")
    o = comm_order(g, zp_compute_order(g))
    assert names(g, o[DISP_LANE]) == ["DispF1,1", "DispF1,2", "DispB1,1", "DispB1,2"]
    assert names(g, o[COMB_LANE]) == ["CombF1,1", "CombF1,2", "CombB1,1", "CombB1,2"]
    g = build_zp_graph(spec(L=3, R=2), dur(), mode="zp-full")
    assert sorted(t for lane in default_orders(g).values() for t in lane) == [t.id for t in g.tasks]


def _fig(**kw):
    base = dict(experts_per_layer=6, layers=3, attention_gpus=1, expert_gpus=1,
                attn_fwd=Fraction(3), single_expert_on_attn=Fraction(3), expert_layer_on_expert=Fraction(4))
    base.update(kw)
    return OffloadPlanInputs(**base)


# test_scheduler.py:139-204 (Algorithm 1, Fig. 4 scenario)
def test_algorithm1_known_answers():
    p = asym_ea_offload(_fig())
    assert p.assignment.offload == (0, 1, 1) and p.t_gather == 1 and p.t_squeeze == Fraction(7, 6)
    assert all(0 <= r < p.t_squeeze for r in p.residuals)
    p = asym_ea_offload(_fig(n_max=1))
    assert p.alpha == Fraction(7, 18) and p.beta == 1 and p.assignment.offload == (0, 0, 1)
    p = asym_ea_offload(_fig(expert_layer_on_expert=Fraction(3)))
    assert p.assignment.offload == (0, 0, 0) and p.note == "no bubbles to squeeze"
    with pytest.raises(InfeasibleError):
        asym_ea_offload(_fig(expert_layer_on_expert=Fraction(2), n_min=1))
    with pytest.raises(InfeasibleError):
        asym_ea_offload(_fig(n_min=3, n_max=1))
    p = asym_ea_offload(_fig(attn_fwd=Fraction(39, 10), n_min=4))
    assert p.beta > 1 and p.assignment.total == 4 and p.residuals[-1] == 0
    v, r = asym_ea_offload(_fig(squeeze_mode="verbatim")), asym_ea_offload(_fig(squeeze_mode="rederived"))
    assert v.t_squeeze == r.t_squeeze and v.assignment == r.assignment
    kw = dict(experts_per_layer=8, attention_gpus=2, expert_gpus=1, single_expert_on_attn=Fraction(2))
    assert asym_ea_offload(_fig(squeeze_mode="verbatim", **kw)).t_squeeze != \
        asym_ea_offload(_fig(squeeze_mode="rederived", **kw)).t_squeeze
    p = asym_ea_offload(_fig(experts_per_layer=8, attention_gpus=2, expert_gpus=1,
                             expert_layer_on_expert=Fraction(6)))
    assert p.chunk[1] == 2 and all(o % 2 == 0 for o in p.assignment.offload)


# test_scheduler.py:208-221
def test_l_busy_and_ledger():
    assert compute_l_busy(4, 3) == 4 and compute_l_busy(2, 1) == 2
    assert compute_l_busy(3, 3) == math.inf and compute_l_busy(2, 5) == math.inf
    ledger = bubble_ledger(OffloadPlanInputs(6, 8, 1, 1, Fraction(3), Fraction(3), Fraction(4)))
    assert ledger[int(compute_l_busy(4, 3)) - 1] == 4


# test_simulator.py:28-54
def test_makespans():
    g = build_zp_graph(spec(L=1, R=1, n=1, k=1, attn=5), dur(attn=5), mode="zp-theorem", include_backward=False)
    assert simulate(g, default_orders(g)).makespan == 5
    g = build_zp_graph(spec(L=1, R=1, n=1, k=1, gamma=Fraction(4, 3)), dur(gamma=Fraction(4, 3)), mode="zp-theorem")
    assert simulate(g, default_orders(g)).makespan == 7
    g = fwd(spec(), dur())
    tl = simulate(g, default_orders(g))
    assert tl.makespan == 39 and validate_timeline(g, tl) == []


# test_simulator.py:57-80
def test_validate_timeline_detects_corruption():
    g = fwd(spec(L=2, R=2), dur())
    tl = simulate(g, default_orders(g))
    bad = Timeline(dict(tl.starts), dict(tl.ends), tl.makespan, tl.lanes)
    a, b = tl.lanes[ATTN_LANE][:2]
    bad.starts[b] = bad.starts[a]
    v = validate_timeline(g, bad)
    assert any("overlaps" in x for x in v) and any("duration" in x for x in v)


# test_simulator.py:112-126
def test_deadlock_and_coverage():
    g = fwd(spec(L=2, R=1), dur())
    o = default_orders(g)
    o[ATTN_LANE] = list(reversed(o[ATTN_LANE]))
    with pytest.raises(DeadlockError) as err:
        simulate(g, o)
    assert len(err.value.cycle) >= 2
    o = default_orders(g)
    o[ATTN_LANE] = o[ATTN_LANE][:-1]
    with pytest.raises(ValueError, match="missing from orders"):
        simulate(g, o)


# test_simulator.py:128-177
def test_metrics_known_answers():
    g = build_zp_graph(spec(L=1, R=2, n=1, k=1, attn=4), dur(attn=4), mode="zp-theorem")
    m = compute_metrics(g, simulate(g, default_orders(g)))
    assert m.devices["attn"].utilization == 1 and m.devices["attn"].bubble_total == 0
    g = fwd(spec(), dur())
    tl = simulate(g, default_orders(g))
    assert compute_metrics(g, tl, tokens_per_iteration=48).throughput_tokens_per_ns == Fraction(48, 39)
    assert bubble_intervals(g, tl, ATTN_LANE) == [(18, 19), (22, 23), (26, 27)]
    g = fwd(spec(L=20, R=3), dur())
    assert abs(float(steady_state_utilization(g, simulate(g, default_orders(g)), "attn", (6, 15))) - 0.75) < 0.02
    s = spec(attn=3000, exp=4000, single=3000)
    d = dur(3000, 4000, 3000)
    zp = fwd(s, d)
    ds = build_distep_graph(s, d, include_backward=False)
    u_zp = compute_metrics(zp, simulate(zp, default_orders(zp))).devices["attn"].utilization_of_makespan
    u_d = compute_metrics(ds, simulate(ds, default_orders(ds))).devices["attn"].utilization_of_makespan
    assert u_d < u_zp


# test_taskgraph.py:60-96
def test_offload_graph_known_answers():
    s = spec(attn=3000, exp=4000, single=3000)
    g = build_zp_graph(s, dur(3000, 4000, 3000), assignment=ExpertAssignment((0, 1, 1)), mode="zp-full")
    assert g.task(TaskKind.EXP_F, 1, 1).duration == 4000
    assert g.task(TaskKind.EXP_F, 2, 1).duration == 3333
    assert g.task(TaskKind.OFF_EXP_F, 2, 1).duration == 500
    assert (g.task(TaskKind.OFF_EXP_F, 2, 1).id, g.task(TaskKind.COMB_F, 2, 1).id) in g.edges
    with pytest.raises(ValidationError):
        build_zp_graph(spec(), dur(), assignment=ExpertAssignment((0, 0, 1)), mode="zp-theorem")
    with pytest.raises(ValidationError):
        build_zp_graph(spec(M=2, N=1), dur(), assignment=ExpertAssignment((0, 1, 0)), mode="zp-full")
    a = ExpertAssignment((0, 1, 2))
    for layer in (1, 2, 3):
        f = token_flow(spec(), a, layer)
        assert f["entering_dispatch"] == f["leaving_combine"]
        assert f["to_expert_gpus"] + f["to_offloaded_experts"] == f["entering_dispatch"]


# test_costmodel.py:75-135
def test_costmodel_known_answers():
    d = derive_task_durations(spec())
    assert (d.attn_fwd, d.expert_layer_fwd_on_expert_gpu, d.single_expert_fwd_on_attn_gpu) == (3, 4, 3)
    fast = GpuClass("fast", 10**12, Fraction(1), Fraction(1, 1000), Fraction(1))
    slow = GpuClass("slow", 10**12, Fraction(1), Fraction(1, 100), Fraction(2))
    cs = Spec(ZpGroupSpec(2, 2, fast, slow, 10**12, 2), ModelSpec(4, 8, 2, 64, 500, 4, 1, 10**6, 0),
              HardwareProfile(fast, slow), RunOptions(gamma=Fraction(1)))
    sh = workload_shape(cs)
    assert sh.tokens_per_microbatch_per_attn_gpu == 500 and sh.tokens_per_expert_gpu == 1000
    assert derive_task_durations(cs).expert_layer_fwd_on_expert_gpu == 2000
    assert derive_task_durations(cs, load_factor=Fraction(3, 2)).expert_layer_fwd_on_expert_gpu == 3000
    assert memory_bounds(spec(expert_mem=10, exp_cap=10**9)).n_min == 0
    assert memory_bounds(spec(L=4, n=24, N=6, M=6, expert_mem=100, exp_cap=1200, attn_cap=10**9)).n_min == 4
    assert memory_bounds(spec(M=2, N=4, n=8, L=2, expert_mem=100, attn_cap=600, exp_cap=10**9)).n_max == 3
    with pytest.raises(InfeasibleError):
        memory_bounds(spec(L=4, n=24, N=6, M=6, expert_mem=100, exp_cap=1200, attn_cap=99))


def test_clamp_to_layer_capacity():
    """Algorithm 1 bounds the offload over all layers, not per layer; the bench clamps each layer
    to whole n_2-chunks within n/N so build_zp_graph accepts the plan (3 + 1: n_2 = 3, n/N = 8)."""
    from paper_2504_03871_b200 import ExpertAssignment
    from paper_2504_03871_b200.planner import clamp_to_layer_capacity

    a, k = clamp_to_layer_capacity(ExpertAssignment((9, 3, 0, 12)), 8, 3, 1)
    assert a.offload == (6, 3, 0, 6) and k == 2
    a, k = clamp_to_layer_capacity(ExpertAssignment((1, 2, 0)), 8, 4, 4)
    assert a.offload == (1, 2, 0) and k == 0
    a, k = clamp_to_layer_capacity(ExpertAssignment((3, 6)), 8, 6, 2)  # n_2 = 3, n/N = 4
    assert a.offload == (3, 3) and k == 1
