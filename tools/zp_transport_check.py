"""Equivalence + timing of the two ZP transports on real GPUs (run under torchrun, 2-8 ranks):
the NCCL send/recv executor (ZpExecutor) and the fused NVLink peer-memory executor
(ZpP2PExecutor) run the same seeded iteration; every gradient must agree, then both are timed.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/zp_transport_check.py [--big]
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2504_03871_b200 import ExpertAssignment, build_zp_graph, derive_task_durations  # noqa: E402
from paper_2504_03871_b200.executor import (NativeBackend, ZpExecutor, ZpLayerShape,  # noqa: E402
                                            ZpP2PExecutor)
from paper_2504_03871_b200.planner import make_zp_spec  # noqa: E402


def grads(ex):
    st = ex.st
    out = {}
    for l in range(1, ex.L + 1):
        for name, t in (("gw_ug", st.gw_ug.get(l)), ("gw_d", st.gw_d.get(l)), ("gwg", st.gwg.get(l)),
                        ("wqkv", st.wqkv[l].grad if l in st.wqkv else None),
                        ("wo", st.wo[l].grad if l in st.wo else None)):
            if t is not None:
                out[f"{name}{l}"] = t.detach().float().clone()
    return out


def fp32_reference(ex, routes, shape, M, seed, dev):
    """Single-process fp32 reference of the executor's iteration (every attention rank's
    micro-batches through the whole L-layer stack), on this rank's GPU: parameters and inputs are
    re-drawn from the executor's seeds (ZpExecutor._init_params), and each (attention rank, layer,
    micro-batch) is routed with the indices that rank's router chose (`routes`), so the comparison
    isolates the executor's data movement and gradients from bf16-vs-fp32 top-k flips (routing
    itself is checked bit-exact against the oracle in test_kernels_gpu / test_parity_gpu).
    Returns the fp32 gradients {name: [layer tensors]}."""
    from paper_2504_03871_b200.executor import attention_block, rms_norm
    from paper_2504_03871_b200.ops import split_gate_up

    s, L, R = shape, ex.L, ex.R
    heads = s.heads or max(1, s.d // 128)
    gen = torch.Generator(device=dev).manual_seed(seed)

    def rand(sh, std):
        return (torch.randn(sh, generator=gen, device=dev) * std).to(torch.bfloat16).float().requires_grad_()

    P = []
    for _ in range(L):
        P.append(dict(wqkv=rand((s.d, 3 * s.d), s.d ** -0.5), wo=rand((s.d, s.d), s.d ** -0.5),
                      wg=rand((s.d, s.E), s.d ** -0.5), w_ug=rand((s.E, 2 * s.f, s.d), s.d ** -0.5),
                      w_d=rand((s.E, s.d, s.f), s.f ** -0.5)))
    for a in range(M):
        g2 = torch.Generator(device=dev).manual_seed(seed * 7919 + 17 + a)
        inputs, gouts = [], []
        for _ in range(R):
            inputs.append(torch.randn((s.tokens_per_mb, s.d), generator=g2, device=dev).to(torch.bfloat16).float())
            gouts.append(torch.randn((s.tokens_per_mb, s.d), generator=g2, device=dev).to(torch.bfloat16).float())
        for j in range(1, R + 1):
            h = inputs[j - 1]
            for l in range(1, L + 1):
                p = P[l - 1]
                u = attention_block(h, p["wqkv"], p["wo"], heads) if s.attention else h * 1
                z = rms_norm(u)
                idx = routes[a][(l, j)].to(dev).long()
                w = torch.softmax(torch.gather(z @ p["wg"], 1, idx), dim=1)
                wgt, wut = split_gate_up(p["w_ug"])
                y = torch.zeros_like(u)
                for slot in range(s.k):
                    for e in range(s.E):
                        m = idx[:, slot] == e
                        if bool(m.any()):
                            ze = z[m]
                            ye = (torch.nn.functional.silu(ze @ wgt[e].t()) * (ze @ wut[e].t())) @ p["w_d"][e].t()
                            y = y.index_add(0, m.nonzero()[:, 0], w[m, slot:slot + 1] * ye)
                h = u + y
            (h * gouts[j - 1]).sum().backward()
    return {name: [p[name].grad.detach() for p in P] for name in ("wqkv", "wo", "wg", "w_ug", "w_d")}


def reference_errors(ex, shape, M, seed, dev):
    """Relative Frobenius error of every gradient of the executor's last iteration (gathered over
    all ranks to rank 0) against fp32_reference; None on ranks != 0."""
    W, rank = dist.get_world_size(), dist.get_rank()
    routes = {key: r.idx.detach().cpu() for key, r in ex.route.items()} if ex.is_attn else {}
    local = {"rank": rank, "routes": routes, "own": ex.st.own,
             "gw_ug": {l: t.detach().float().cpu() for l, t in ex.st.gw_ug.items()},
             "gw_d": {l: t.detach().float().cpu() for l, t in ex.st.gw_d.items()},
             "gwg": {l: t.detach().float().cpu() for l, t in ex.st.gwg.items()},
             "wqkv": {l: t.grad.detach().float().cpu() for l, t in ex.st.wqkv.items() if t.grad is not None},
             "wo": {l: t.grad.detach().float().cpu() for l, t in ex.st.wo.items() if t.grad is not None}}
    allv = [None] * W
    dist.all_gather_object(allv, local)
    if rank != 0:
        return None
    allv.sort(key=lambda o: o["rank"])
    ref = fp32_reference(ex, [allv[a]["routes"] for a in range(M)], shape, M, 5, dev)
    errs = {}
    for l in range(1, ex.L + 1):
        g_ug = torch.zeros_like(ref["w_ug"][l - 1]).cpu()
        g_d = torch.zeros_like(ref["w_d"][l - 1]).cpu()
        for o in allv:
            own = o["own"][l - 1]
            if own:
                g_ug[own] += o["gw_ug"][l]
                g_d[own] += o["gw_d"][l]
        got = {"w_ug": g_ug, "w_d": g_d,
               "wg": sum(o["gwg"][l] for o in allv if l in o["gwg"]),
               "wqkv": sum(o["wqkv"][l] for o in allv if l in o["wqkv"]),
               "wo": sum(o["wo"][l] for o in allv if l in o["wo"])}
        for name, g in got.items():
            r_ = ref[name][l - 1].cpu()
            errs[f"{name}{l}"] = float((g - r_).norm() / r_.norm().clamp_min(1e-30))
    return errs


def zero_attn_grads(ex):
    for d in (ex.st.wqkv, ex.st.wo):
        for t in d.values():
            t.grad = None


def timed(ex, iters):
    ex.run()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        ex.run()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def main():
    if os.environ.get("HM_DUMP_AFTER"):  # debugging a hang: dump every thread's stack, then exit
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["HM_DUMP_AFTER"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="C2 shapes (d=4096, f=14336)")
    ap.add_argument("--offload", default="",
                    help="experts offloaded per expert rank: one value for every layer, or one per layer")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--ref", action="store_true",
                    help="also compare both transports' gradients with a single-process fp32 stack")
    args = ap.parse_args()
    os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")
    # attention backward (SDPA) may accumulate with atomics; the check wants run-to-run
    # determinism so that any difference is the transport's
    torch.use_deterministic_algorithms(True, warn_only=True)
    dist.init_process_group("nccl")
    W, rank = dist.get_world_size(), dist.get_rank()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    M = W // 2
    N = W - M
    if args.big:
        E, k, d, f, T, L, R = 8, 2, 4096, 14336, 2048, 2, 4
    else:
        E, k, d, f, T, L, R = 8, 2, 512, 512, 512, 2, 3
    if args.offload:
        off = [int(v) for v in args.offload.split(",")]
        off = off * L if len(off) == 1 else off
    else:
        off = [1 if E // N > 1 else 0] * L
    spec = make_zp_spec(M, N, L, R, E, k, T, d, attn_fwd_ns=3000, expert_layer_fwd_ns=4000,
                        single_expert_fwd_ns=3000, dispatch_ns=100, combine_ns=100)
    graph = build_zp_graph(spec, derive_task_durations(spec), ExpertAssignment(tuple(off)),
                           mode="zp-full")
    shape = ZpLayerShape(E, k, d, f, T)
    disp = dist.new_group(list(range(W)))
    comb = dist.new_group(list(range(W)))
    be = NativeBackend(dev)
    results = {}
    ex_n = ZpExecutor(graph, shape, M, N, rank, be, disp, comb, seed=5)
    ex_n.run()
    torch.cuda.synchronize()
    g_n = grads(ex_n)
    zero_attn_grads(ex_n)
    ex_n.run()  # run-to-run noise floor of the NCCL executor itself
    torch.cuda.synchronize()
    self_rel = max(float((a - b).norm() / a.norm().clamp_min(1e-30)) for a, b in
                   zip(g_n.values(), grads(ex_n).values()))
    ref_errs = {}
    if args.ref:
        torch.backends.cuda.matmul.allow_tf32 = False
        ref_errs["nccl"] = reference_errors(ex_n, shape, M, 5, dev)
    ex_p = ZpP2PExecutor(graph, shape, M, N, rank, be, disp, comb, seed=5)
    worst = 0.0
    for it in range(2):  # the second iteration re-uses the arena and the monotonic flags
        zero_attn_grads(ex_p)
        ex_p.run()
        torch.cuda.synchronize()
        g_p = grads(ex_p)
        for key, a in g_n.items():
            b = g_p[key]
            rel = float((a - b).norm() / a.norm().clamp_min(1e-30))
            worst = max(worst, rel)
            if it == 0:
                results[key] = {"rel": rel, "bitwise": bool(torch.equal(a, b))}
    if args.ref:
        ref_errs["p2p"] = reference_errors(ex_p, shape, M, 5, dev)
    zero_attn_grads(ex_n)
    zero_attn_grads(ex_p)
    ms_n = timed(ex_n, args.iters)
    ms_p = timed(ex_p, args.iters)
    wt = torch.tensor([worst, self_rel], device=dev)
    dist.all_reduce(wt, op=dist.ReduceOp.MAX)
    worst, self_rel = float(wt[0]), float(wt[1])
    if rank == 0:
        print(json.dumps({"world": W, "M": M, "N": N, "shape": [E, k, d, f, T, L, R], "offload": off,
                          "worst_rel_err": worst, "nccl_rerun_rel_err": self_rel, "rank0": results,
                          "ms_per_iter": {"nccl": ms_n, "p2p": ms_p},
                          "vs_fp32_reference": ref_errs or None}))
    dist.barrier()
    dist.destroy_process_group()
    if worst > max(1e-3, 4 * self_rel):
        sys.exit(1)


if __name__ == "__main__":
    main()
