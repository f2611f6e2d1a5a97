"""B200 profiler -> planner loop (the paper's Profiler).

Measures, on the local GPU, the per-micro-batch forward times the planner needs and returns
them as the reference's duration table (``profile.attention_gpu.durations`` /
``profile.expert_gpu.durations`` / ``profile.comm``, ``core.py:269-300``), which
``derive_task_durations`` prefers over coefficients (``costmodel.py:88-104``):

  attn_fwd             attention block + router + dispatch permute of one micro-batch
  expert_layer_fwd     grouped SwiGLU FFN of the B = s*M*k/N rows an expert rank receives,
                       over its E/N experts, with the rank's capacity cap (max_ctas)
  single_expert_fwd    one expert over B rows on an attention GPU
  dispatch / combine   one (layer, micro-batch) exchange, timed on the real communicator
                       (``measure_exchange``: NCCL all-to-all with the ZP split sizes)

and the memory side of the paper's profiler (``PAPER.md:364``; the reference turns it into
offload bounds in ``costmodel.memory_bounds``, ``costmodel.py:124-161``): ``measure_memory``
measures bytes per expert (weights + the executor's fp32 gradient accumulators), the activation
bytes an expert rank keeps per routed row and an attention rank per token and layer, attention
parameters per layer, and the device capacity, which ``memory_spec_fields`` folds into the
spec's ``expert_mem`` / ``memory_capacity`` / ``non_expert_mem_*`` fields.
"""

from __future__ import annotations

from typing import Optional

import torch

NVLINK_GBS = 770.0  # peer copy bandwidth per direction (B200_PROFILING.md); fallback only


def _time_ms(fn, reps: int = 5, warmup: int = 2) -> float:
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def measure_loads(shape, device="cuda", seed: int = 0) -> list:
    """Routed rows per expert for one micro-batch (attention block, pre-norm, router with the
    config's logit bias): the expected expert loads for a skew-aware placement."""
    from . import ops
    from .executor import attention_block, rms_norm

    dev = torch.device(device)
    g = torch.Generator(device=dev).manual_seed(seed)
    d, E, k, T = shape.d, shape.E, shape.k, shape.tokens_per_mb
    heads = shape.heads or max(1, d // 128)
    rnd = lambda *s, std=1.0: (torch.randn(s, generator=g, device=dev) * std).to(torch.bfloat16)  # noqa: E731
    x = rnd(T, d)
    wqkv, wo, wg = rnd(d, 3 * d, std=d ** -0.5), rnd(d, d, std=d ** -0.5), rnd(d, E, std=d ** -0.5)
    bias = None
    if getattr(shape, "router_skew", 0.0):
        from .configs import zipf_bias

        bias = torch.tensor(zipf_bias(E, shape.router_skew), dtype=torch.float32, device=dev)
    u = attention_block(x, wqkv, wo, heads) if shape.attention else x
    r = ops.router_topk(rms_norm(u), wg, k, bias)
    return [int(c) for c in r.counts.tolist()]


def measure_durations(shape, M: int, N: int, expert_max_ctas: int = 0, attn_max_ctas: int = 0,
                      device="cuda", seed: int = 0, loads=None, capacity=None, microbatches: int = 8,
                      balance_roles: bool = True) -> dict:
    """Duration table (ns) for ``planner.make_zp_spec`` measured with the native kernels.
    With ``loads`` (``measure_loads``) the expert layer is timed on the busiest expert rank of
    the load-balanced placement (the reference's ``load_factor`` for skew, costmodel.py:54-63),
    with that rank's real per-expert row counts; with per-rank ``capacity`` weights the busiest
    rank is the one with the largest load / capacity, and ``expert_max_ctas`` should be that
    rank's grid cap (the caller passes the slowest rank's).

    Backward: the reference prices every backward task at gamma x its forward (one gamma for all
    kinds, ``core.py:113-122``). gamma is measured on the expert layer as the executor runs it
    (data gradients per micro-batch, the layer's weight gradients once over ``microbatches``
    micro-batches, so 1/R of that launch per micro-batch). The attention rank's backward (router
    backward, attention + pre-norm autograd, combine backward) has a larger ratio on B200 (~3 vs
    ~2), so with ``balance_roles`` the attention forward handed to the planner is normalised to
    (fwd + bwd) / (1 + gamma): its forward + backward total is the measured one and Algorithm 1
    balances the roles on their real per-micro-batch work. The raw times are returned beside it."""
    from . import ops
    from .executor import attention_block, rms_norm

    dev = torch.device(device)
    g = torch.Generator(device=dev).manual_seed(seed)
    d, f, E, k, T = shape.d, shape.f, shape.E, shape.k, shape.tokens_per_mb
    heads = shape.heads or max(1, d // 128)

    def rnd(*s, std=1.0):
        return (torch.randn(s, generator=g, device=dev) * std).to(torch.bfloat16)

    x = rnd(T, d)
    wqkv, wo, wg = rnd(d, 3 * d, std=d ** -0.5), rnd(d, d, std=d ** -0.5), rnd(d, E, std=d ** -0.5)
    bias = None
    if getattr(shape, "router_skew", 0.0):
        from .configs import zipf_bias

        bias = torch.tensor(zipf_bias(E, shape.router_skew), dtype=torch.float32, device=dev)

    def attn_step():
        u = attention_block(x, wqkv, wo, heads) if shape.attention else x
        z = rms_norm(u)
        r = ops.router_topk(z, wg, k, bias)
        ops.dispatch_permute(z, r)

    attn_ms = _time_ms(attn_step)
    # the attention rank's backward of one micro-batch, as ATTN_B / DISP_B run it
    wqkv_p, wo_p = wqkv.clone().requires_grad_(), wo.clone().requires_grad_()
    wg_t = ops.transpose_bf16(wg)
    y_perm, dxp, dh_out = rnd(T * k, d), rnd(T * k, d), rnd(T, d)

    def attn_fwd_bwd():
        hh = x.detach().requires_grad_()
        with torch.enable_grad():
            u = attention_block(hh, wqkv_p, wo_p, heads) if shape.attention else hh * 1
            z = rms_norm(u)
        zd = z.detach()
        r = ops.router_topk(zd, wg, k, bias)
        xp, _, row_of = ops.dispatch_permute(zd, r)
        _dy_perm, dw = ops.combine_bwd(dh_out, y_perm, row_of, r.w)
        dz, _dl, _dwg = ops.router_bwd(dxp, row_of, r, dw, xp, wg_t, want_dwg=True, x=zd)
        torch.autograd.backward([u, z], [dh_out, dz.to(z.dtype)])

    attn_bwd_ms = max(_time_ms(attn_fwd_bwd) - attn_ms, 0.0)

    B = T * M * k // N
    e_local = E // N
    seg_l = [B * i // e_local for i in range(e_local + 1)]
    if loads is not None:
        from .executor import expert_owners

        owners = expert_owners(E, M, N, 0, loads, capacity)
        tot = sum(loads)
        cap = list(capacity) if capacity is not None else [1.0] * N
        per_rank = [[e for e in range(E) if owners[e] == M + i] for i in range(N)]
        busiest = max(range(N), key=lambda i: sum(loads[e] for e in per_rank[i]) / cap[i])
        busiest = per_rank[busiest]
        rows = [T * M * k * loads[e] // tot for e in busiest]
        seg_l = [0]
        for r_ in rows:
            seg_l.append(seg_l[-1] + r_)
        B = seg_l[-1]
    w_ug = rnd(max(e_local, 1), 2 * f, d, std=d ** -0.5)
    w_d = rnd(max(e_local, 1), d, f, std=f ** -0.5)
    xb = rnd(B, d)
    seg = torch.tensor(seg_l, dtype=torch.int32, device=dev)
    exp_ms = _time_ms(lambda: ops.grouped_ffn_fwd(xb, seg, w_ug, w_d, expert_max_ctas))
    B1 = T * M * k // N // max(e_local, 1) * e_local  # an offloaded expert: average share
    seg1 = torch.tensor([0, min(B1, B)], dtype=torch.int32, device=dev)
    single_ms = _time_ms(lambda: ops.grouped_ffn_fwd(xb, seg1, w_ug[:1].contiguous(), w_d[:1].contiguous(),
                                                     attn_max_ctas))
    # backward factor gamma: the expert layer's backward as the executor runs it (data gradients
    # per micro-batch + 1/R of the layer's once-per-layer weight-gradient launch) / forward
    y, h, act = ops.grouped_ffn_fwd(xb, seg, w_ug, w_d, expert_max_ctas)
    gw_ug = torch.zeros(w_ug.shape, dtype=torch.float32, device=dev)
    gw_d = torch.zeros(w_d.shape, dtype=torch.float32, device=dev)
    data_ms = _time_ms(lambda: ops.grouped_ffn_bwd_data(y, xb, h, act, seg, w_ug, w_d, expert_max_ctas))
    _dx, dh = ops.grouped_ffn_bwd_data(y, xb, h, act, seg, w_ug, w_d, expert_max_ctas)
    R = max(1, int(microbatches))
    seg_multi = seg.view(1, -1).repeat(R, 1).contiguous()

    def wgrad_layer():
        ops.grouped_wgrad_multi([dh] * R, [xb] * R, seg_multi, gw_ug, max_ctas=expert_max_ctas)
        ops.grouped_wgrad_multi([y] * R, [act] * R, seg_multi, gw_d, max_ctas=expert_max_ctas)

    bwd_ms = data_ms + _time_ms(wgrad_layer, reps=2, warmup=1) / R
    gamma = bwd_ms / exp_ms
    attn_plan_ms = (attn_ms + attn_bwd_ms) / (1.0 + gamma) if balance_roles else attn_ms
    comm_ns = T * k * d * 2 / (NVLINK_GBS * 1e9) * 1e9
    return {
        "gamma_x100": int(round(100 * gamma)),
        "attn_fwd_ns": int(attn_plan_ms * 1e6),
        "expert_layer_fwd_ns": int(exp_ms * 1e6),
        "single_expert_fwd_ns": int(single_ms * 1e6),
        "dispatch_ns": int(comm_ns),
        "combine_ns": int(comm_ns),
        # measured, for the record (not planner inputs)
        "attn_fwd_measured_ns": int(attn_ms * 1e6),
        "attn_bwd_measured_ns": int(attn_bwd_ms * 1e6),
        "expert_layer_bwd_measured_ns": int(bwd_ms * 1e6),
    }


PLANNER_DURATION_KEYS = ("attn_fwd_ns", "expert_layer_fwd_ns", "single_expert_fwd_ns", "dispatch_ns", "combine_ns")


def measure_memory(shape, device="cuda", seed: int = 0) -> dict:
    """Memory probe with the native kernels on this GPU. Returns bytes:

      capacity              total device memory (cudaMemGetInfo)
      outside_torch         memory in use that torch did not allocate (CUDA context, NCCL)
      expert_mem            one expert: bf16 W_ug + W_d and the fp32 gradient accumulators the
                            executor keeps per owned expert (optimizer state is not held)
      expert_act_per_row    what an expert rank keeps per routed row and layer between the
                            forward and the backward (y, h, act of the grouped FFN)
      attn_act_per_token    what an attention rank keeps per token and layer (attention block
                            autograd state, pre-norm input, routing, permuted rows)
      attn_params_per_layer attention block + router weights of one layer and their gradients
    """
    from . import ops
    from .executor import attention_block, rms_norm

    dev = torch.device(device)
    torch.cuda.synchronize(dev)
    free, total = torch.cuda.mem_get_info(dev)
    outside = total - free - torch.cuda.memory_reserved(dev)
    g = torch.Generator(device=dev).manual_seed(seed)
    d, f, E, k, T = shape.d, shape.f, shape.E, shape.k, shape.tokens_per_mb
    heads = shape.heads or max(1, d // 128)

    def rnd(*s, std=1.0):
        return (torch.randn(s, generator=g, device=dev) * std).to(torch.bfloat16)

    def alloc():
        torch.cuda.synchronize(dev)
        return torch.cuda.memory_allocated(dev)

    m0 = alloc()
    w_ug = rnd(1, 2 * f, d, std=d ** -0.5)
    w_d = rnd(1, d, f, std=f ** -0.5)
    gw_ug = torch.zeros(w_ug.shape, dtype=torch.float32, device=dev)
    gw_d = torch.zeros(w_d.shape, dtype=torch.float32, device=dev)
    expert_mem = alloc() - m0

    rows = max(T * k // max(E, 1), 256)  # one expert's share of a micro-batch
    xb = rnd(rows, d)
    seg = torch.tensor([0, rows], dtype=torch.int32, device=dev)
    m1 = alloc()
    kept = ops.grouped_ffn_fwd(xb, seg, w_ug, w_d)
    expert_act = (alloc() - m1) / rows
    del kept, xb, w_ug, w_d, gw_ug, gw_d

    m2 = alloc()
    wqkv = rnd(d, 3 * d, std=d ** -0.5).requires_grad_()
    wo = rnd(d, d, std=d ** -0.5).requires_grad_()
    wg = rnd(d, E, std=d ** -0.5)
    attn_params = 2 * (alloc() - m2) + d * E * 4  # + their gradients (same size) + fp32 router grad
    x = rnd(T, d).requires_grad_()
    m3 = alloc()
    with torch.enable_grad():
        u = attention_block(x, wqkv, wo, heads) if shape.attention else x * 1
        z = rms_norm(u)
    r = ops.router_topk(z.detach(), wg, k)
    x_perm, _, row_of = ops.dispatch_permute(z.detach(), r)
    attn_act = (alloc() - m3) / T
    del u, z, r, x_perm, row_of, x, wqkv, wo, wg
    torch.cuda.empty_cache()
    return {"capacity": int(total), "outside_torch": int(max(outside, 0)), "expert_mem": int(expert_mem),
            "expert_act_per_row": int(round(expert_act)), "attn_act_per_token": int(round(attn_act)),
            "attn_params_per_layer": int(attn_params)}


def memory_spec_fields(mem: dict, M: int, N: int, layers: int, microbatches: int, tokens_per_mb: int,
                       k: int, arena_bytes: int = 0) -> dict:
    """The measured probe as the reference's memory model (``costmodel.memory_bounds``): per role,
    ``non_expert_mem_*`` = memory outside torch + the transport arena + the activations resident
    at the ZP peak (all L layers x R micro-batches in flight before the first backward) + (attention)
    its parameters; ``activation_mem_per_token`` stays 0 because the per-role activation bytes
    differ and are folded into the per-role terms."""
    rows_per_mb = tokens_per_mb * M * k // N  # routed rows one expert rank receives (R6's B)
    exp_non = mem["outside_torch"] + arena_bytes + mem["expert_act_per_row"] * rows_per_mb * microbatches * layers
    attn_non = (mem["outside_torch"] + arena_bytes + mem["attn_params_per_layer"] * layers
                + mem["attn_act_per_token"] * tokens_per_mb * microbatches * layers)
    return {"expert_mem": mem["expert_mem"], "attn_capacity": mem["capacity"], "exp_capacity": mem["capacity"],
            "non_expert_mem_attention": int(attn_non), "non_expert_mem_expert": int(exp_non)}


def measure_exchange(M: int, N: int, tokens_per_mb: int, k: int, d: int, group=None, reps: int = 5) -> int:
    """One (layer, micro-batch) dispatch exchange timed on the real communicator (collective: every
    rank calls it): each attention rank sends tokens_per_mb*k/N routed bf16 rows to every expert
    rank through NCCL all_to_all_single with the ZP split sizes (the combine is the mirror
    image). CUDA events, max over ranks, ns."""
    import torch.distributed as dist

    W = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = tokens_per_mb * k // N
    send = [per if (rank < M and q >= M) else 0 for q in range(W)]
    recv = [per if (rank >= M and q < M) else 0 for q in range(W)]
    dev = torch.device("cuda", torch.cuda.current_device())
    sb = torch.empty((max(sum(send), 1), d), dtype=torch.bfloat16, device=dev)
    rb = torch.empty((max(sum(recv), 1), d), dtype=torch.bfloat16, device=dev)

    def once():
        dist.all_to_all_single(rb[: sum(recv)], sb[: sum(send)], recv, send, group=group)

    once()
    torch.cuda.synchronize(dev)
    dist.barrier(group=group)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        once()
    b.record()
    torch.cuda.synchronize(dev)
    t = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(float(t) * 1e6)


def measure_transport(shape, M: int, N: int, backend, transport: str = "p2p", disp_group=None,
                      comb_group=None, reps: int = 3, seed: int = 11) -> dict:
    """The exchange as the executor performs it (collective: every rank calls it): a one-layer,
    one-micro-batch ZP graph (no offload) run through the real executor (``ZpP2PExecutor`` /
    ``ZpExecutor``) with the chosen transport, each exchange timed on its SENDING role — DISP_F on
    the attention ranks (count all-gather, the permute with its peer stores, the completion
    flags), COMB_F on the expert ranks (the return is fused into the down-projection GEMM, so
    with peer memory this is only the flag release; with NCCL the send) — median over ``reps``
    iterations, max over the role's ranks, in ns. (The receiving side's interval would also
    contain the wait for the other role's compute.) These are the planner's ``dispatch`` /
    ``combine`` entries (the reference prices them as bytes / bandwidth, ``costmodel.py:40-47``)."""
    import statistics

    import torch.distributed as dist

    from .core import ExpertAssignment
    from .costmodel import derive_task_durations
    from .executor import ZpExecutor, ZpP2PExecutor, execute
    from .planner import make_zp_spec
    from .taskgraph import TaskKind, build_zp_graph

    spec = make_zp_spec(M, N, 1, 1, shape.E, shape.k, shape.tokens_per_mb, shape.d, attn_fwd_ns=1000,
                        expert_layer_fwd_ns=1000, single_expert_fwd_ns=1000, dispatch_ns=100, combine_ns=100)
    graph = build_zp_graph(spec, derive_task_durations(spec), ExpertAssignment((0,)), mode="zp-full")
    cls = ZpP2PExecutor if transport == "p2p" else ZpExecutor
    ex = cls(graph, shape, M, N, dist.get_rank(), backend, disp_group, comb_group, seed=seed)
    ex.run()  # warm-up
    samples = {"DispF": [], "CombF": []}
    for _ in range(reps):
        tl = execute(graph, ex)
        for t in graph.tasks:
            if t.kind in (TaskKind.DISP_F, TaskKind.COMB_F):
                senders = range(M) if t.kind == TaskKind.DISP_F else range(M, M + N)
                ds = [tl.per_rank[r][t.id][1] - tl.per_rank[r][t.id][0] for r in senders if t.id in tl.per_rank[r]]
                samples[t.kind.value].append(max(ds))
    out = {k: int(statistics.median(v)) for k, v in samples.items()}
    del ex
    torch.cuda.empty_cache()
    return {"dispatch_ns": out["DispF"], "combine_ns": out["CombF"]}


def calibrate_in_pipeline(shape, M: int, N: int, backend, offload, transport: str = "p2p",
                          disp_group=None, comb_group=None, microbatches: int = 8, reps: int = 2,
                          expert_loads=None, expert_capacity=None, base: Optional[dict] = None,
                          seed: int = 13) -> dict:
    """Planner durations measured INSIDE the pipeline (collective: every rank calls it).

    The isolated probes of ``measure_durations`` run at burst clocks and without the exchange
    kernels beside them; in the pipeline every task runs at sustained-power clocks, and under a
    skewed router the busiest expert rank and the offloaded experts carry other loads than one
    routed micro-batch suggests. This runs a ``len(offload)``-layer ZP graph with the given
    per-layer offloads and ``microbatches`` micro-batches through the real executor and inverts the
    reference's duration model (``taskgraph.py:253-263``: ExpF = T_exp·(1 − o·N/n),
    OffExpF = T_single·o·N²/(n·M), backward = γ × forward) on the measured tasks, each task's
    duration taken as the max over its role's ranks and averaged over micro-batches and layers.
    Returns the planner's duration keys (``attn_fwd_ns`` normalised to (fwd + bwd) / (1 + γ) as in
    ``measure_durations``); ``single_expert_fwd_ns`` falls back to ``base`` scaled by the measured /
    profiled expert-layer ratio when no calibration layer offloads."""
    import torch.distributed as dist

    from .core import ExpertAssignment
    from .costmodel import derive_task_durations
    from .executor import ZpExecutor, ZpP2PExecutor, execute
    from .planner import make_zp_spec
    from .taskgraph import TaskKind, build_zp_graph

    L = len(offload)
    n = shape.E
    spec = make_zp_spec(M, N, L, microbatches, shape.E, shape.k, shape.tokens_per_mb, shape.d,
                        attn_fwd_ns=1000, expert_layer_fwd_ns=1000, single_expert_fwd_ns=1000,
                        dispatch_ns=100, combine_ns=100)
    graph = build_zp_graph(spec, derive_task_durations(spec), ExpertAssignment(tuple(offload)), mode="zp-full")
    cls = ZpP2PExecutor if transport == "p2p" else ZpExecutor
    ex = cls(graph, shape, M, N, dist.get_rank(), backend, disp_group, comb_group, seed=seed,
             expert_loads=expert_loads, expert_capacity=expert_capacity)
    ex.run()
    ex.run()  # warm-up: sustained clocks before the measured iterations
    acc = {}
    for _ in range(reps):
        tl = execute(graph, ex)
        for t in graph.tasks:
            role = range(0, M) if t.device == "attn" else range(M, M + N)
            ds = [tl.per_rank[r][t.id][1] - tl.per_rank[r][t.id][0] for r in role if t.id in tl.per_rank[r]]
            if ds:
                acc.setdefault((t.kind, t.layer), []).append(max(ds))
    del ex
    torch.cuda.empty_cache()
    mean = lambda v: sum(v) / len(v)  # noqa: E731
    kind = lambda kd: [mean(v) for (k_, l_), v in acc.items() if k_ == kd]  # noqa: E731
    attn_f, attn_b = mean(kind(TaskKind.ATTN_F)), mean(kind(TaskKind.ATTN_B))
    t_exp, t_exp_b, t_single = [], [], []
    for (k_, l_), v in acc.items():
        o = offload[l_ - 1]
        if k_ in (TaskKind.EXP_F, TaskKind.EXP_B) and o * N < n:
            (t_exp if k_ == TaskKind.EXP_F else t_exp_b).append(mean(v) / (1 - o * N / n))
        if k_ == TaskKind.OFF_EXP_F and o > 0:
            t_single.append(mean(v) / (o * N * N / (n * M)))
    if not t_exp or not t_exp_b:  # every calibration layer offloaded all experts: keep the probe's
        if not base:
            raise ValueError("calibrate_in_pipeline: no expert-rank task to invert and no base durations")
        exp_f = base["expert_layer_fwd_ns"] * (mean(kind(TaskKind.ATTN_F)) / base["attn_fwd_measured_ns"]
                                               if base.get("attn_fwd_measured_ns") else 1.0)
        gamma = base["gamma_x100"] / 100
    else:
        exp_f = mean(t_exp)
        gamma = mean(t_exp_b) / exp_f
    if t_single:
        single = mean(t_single)
    elif base:
        single = base["single_expert_fwd_ns"] * exp_f / base["expert_layer_fwd_ns"]
    else:
        single = exp_f * N / n
    return {"attn_fwd_ns": int((attn_f + attn_b) / (1 + gamma)), "expert_layer_fwd_ns": int(exp_f),
            "single_expert_fwd_ns": int(single), "gamma_x100": int(round(100 * gamma)),
            "attn_fwd_raw_ns": int(attn_f), "attn_bwd_raw_ns": int(attn_b)}
