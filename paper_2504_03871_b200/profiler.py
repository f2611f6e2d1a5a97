"""B200 profiler -> planner loop (the paper's Profiler).

Measures, on the local GPU, the per-micro-batch forward times the planner needs and returns
them as the reference's duration table (``profile.attention_gpu.durations`` /
``profile.expert_gpu.durations`` / ``profile.comm``, ``core.py:269-300``), which
``derive_task_durations`` prefers over coefficients (``costmodel.py:88-104``):

  attn_fwd             attention block + router + dispatch permute of one micro-batch
  expert_layer_fwd     grouped SwiGLU FFN of the B = s*M*k/N rows an expert rank receives,
                       over its E/N experts, with the rank's capacity cap (max_ctas)
  single_expert_fwd    one expert over B rows on an attention GPU
  dispatch / combine   bytes per attention rank over the measured NVLink peer bandwidth
"""

from __future__ import annotations

import torch

NVLINK_GBS = 770.0  # measured peer copy bandwidth per direction (B200_PROFILING.md)


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
                      device="cuda", seed: int = 0, loads=None) -> dict:
    """Duration table (ns) for ``planner.make_zp_spec`` measured with the native kernels.
    With ``loads`` (``measure_loads``) the expert layer is timed on the busiest expert rank of
    the load-balanced placement (the reference's ``load_factor`` for skew, costmodel.py:54-63),
    with that rank's real per-expert row counts."""
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

    B = T * M * k // N
    e_local = E // N
    seg_l = [B * i // e_local for i in range(e_local + 1)]
    if loads is not None:
        from .executor import expert_owners

        owners = expert_owners(E, M, N, 0, loads)
        tot = sum(loads)
        per_rank = [[e for e in range(E) if owners[e] == M + i] for i in range(N)]
        busiest = max(per_rank, key=lambda es: sum(loads[e] for e in es))
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
    # backward factor gamma: the expert layer's measured backward / forward time (the reference
    # applies one gamma to every task kind, core.py:113-122)
    y, h, act = ops.grouped_ffn_fwd(xb, seg, w_ug, w_d, expert_max_ctas)
    gw_ug = torch.zeros(w_ug.shape, dtype=torch.float32, device=dev)
    gw_d = torch.zeros(w_d.shape, dtype=torch.float32, device=dev)
    bwd_ms = _time_ms(lambda: ops.grouped_ffn_bwd_acc(y, xb, h, act, seg, w_ug, w_d, gw_ug, gw_d,
                                                      expert_max_ctas))
    comm_ns = T * k * d * 2 / (NVLINK_GBS * 1e9) * 1e9
    return {
        "gamma_x100": int(round(100 * bwd_ms / exp_ms)),
        "attn_fwd_ns": int(attn_ms * 1e6),
        "expert_layer_fwd_ns": int(exp_ms * 1e6),
        "single_expert_fwd_ns": int(single_ms * 1e6),
        "dispatch_ns": int(comm_ns),
        "combine_ns": int(comm_ns),
    }
