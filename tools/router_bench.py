"""Router forward / backward timing on one config (GPU box): K1 (logits + top-k + scan) and the
router backward with the token-major and the permuted-row weight-gradient kernels, interleaved.

    python tools/router_bench.py [C2|C3] [--reps 30]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_layer_tensors  # noqa: E402
from paper_2504_03871_b200 import ops  # noqa: E402
from paper_2504_03871_b200.configs import CONFIGS  # noqa: E402


_BUSY = None


def timed(fn, reps, inner=10):
    """Median over `reps` of the device time of `inner` back-to-back calls, each batch queued
    behind a ~5 ms matmul so host launch overhead never starves the GPU."""
    global _BUSY
    if _BUSY is None:
        _BUSY = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        for _ in range(4):
            _BUSY @ _BUSY
        a.record()
        for _ in range(inner):
            fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / inner)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("--reps", type=int, default=30)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    x, wg, w_ug, w_d, dy = make_layer_tensors(cfg, 1, torch.device("cuda"))
    r = ops.router_topk(x, wg, cfg.k)
    xp, _, row_of = ops.dispatch_permute(x, r)
    dxp = torch.randn_like(xp)
    dw = torch.randn_like(r.w)
    wg_t = ops.transpose_bf16(wg)
    T, d, E, k = cfg.T, cfg.d, cfg.E, cfg.k
    out = {"config": args.config}
    fw = {}
    for variant in ("fused", "unfused", "fused", "unfused"):
        if variant == "unfused":
            os.environ["HM_ROUTER_UNFUSED"] = "1"
        else:
            os.environ.pop("HM_ROUTER_UNFUSED", None)
        fw.setdefault(variant, []).append(timed(lambda: ops.router_topk(x, wg, k), args.reps))
    os.environ.pop("HM_ROUTER_UNFUSED", None)
    # top-k kernel: thread-per-token (default, E <= 64) vs warp-per-token (HM_TOPK_WARP), on the
    # unfused path, every routing output compared bitwise (incl. ties and a NaN/-inf row)
    xt = x.clone()
    xt[1] = 0  # all-zero logits: every expert ties
    xt[2] = float("nan")
    os.environ["HM_ROUTER_UNFUSED"] = "1"
    rt = {}
    for variant in ("lane", "warp", "lane", "warp"):
        if variant == "warp":
            os.environ["HM_TOPK_WARP"] = "1"
        else:
            os.environ.pop("HM_TOPK_WARP", None)
        fw.setdefault("unfused_topk_" + variant, []).append(timed(lambda: ops.router_topk(x, wg, k), args.reps))
        rr = ops.router_topk(xt, wg, k)
        rt[variant] = [rr.idx, rr.w, rr.counts, rr.offsets, rr.chunk_base]
    os.environ.pop("HM_TOPK_WARP", None)
    os.environ.pop("HM_ROUTER_UNFUSED", None)
    bits = [(a.view(torch.int32) if a.dtype == torch.float32 else a) for a in rt["lane"]]
    bits_w = [(a.view(torch.int32) if a.dtype == torch.float32 else a) for a in rt["warp"]]
    out["topk_lane_bitwise_equal"] = {n: bool(torch.equal(a, b)) for n, a, b in
                                      zip(("idx", "w", "counts", "offsets", "chunk_base"), bits, bits_w)}
    out["router_fwd_ms_variants"] = {v: min(t) for v, t in fw.items()}
    out["router_fwd_ms"] = min(fw["fused"])
    res = {}
    envs = {"fused": "HM_ROUTER_BWD_FUSED", "stream": None, "tok": "HM_ROUTER_WGRAD_TOK",
            "perm": "HM_ROUTER_WGRAD_PERM"}
    for variant in ("fused", "stream", "tok", "perm") * 2:
        for e_ in envs.values():
            if e_:
                os.environ.pop(e_, None)
        if envs[variant]:
            os.environ[envs[variant]] = "1"
        ms = timed(lambda: ops.router_bwd(dxp, row_of, r, dw, xp, wg_t, want_dwg=True, x=x), args.reps)
        res.setdefault(variant, []).append(ms)
        res.setdefault(variant + "_dwg", ops.router_bwd(dxp, row_of, r, dw, xp, wg_t, want_dwg=True, x=x)[2].float())
    for e_ in envs.values():
        if e_:
            os.environ.pop(e_, None)
    out["router_bwd_ms"] = {v: min(res[v]) for v in envs}
    out["dwg_rel_diff_stream_vs_perm"] = float((res["stream_dwg"] - res["perm_dwg"]).norm() / res["perm_dwg"].norm())
    # unpermute + dlogit.Wg kernel variants (HM_UNPERMUTE_V1/V2/V3), dx / dlogit compared bitwise
    uv = {}
    for variant in ("v1", "v2", "v3", "v1", "v2", "v3"):
        for v in ("V1", "V2", "V3"):
            os.environ.pop("HM_UNPERMUTE_" + v, None)
        os.environ["HM_UNPERMUTE_" + variant.upper()] = "1"
        uv.setdefault(variant, []).append(timed(lambda: ops.router_bwd(dxp, row_of, r, dw, xp, wg_t, want_dwg=False), args.reps))
        uv.setdefault(variant + "_out", ops.router_bwd(dxp, row_of, r, dw, xp, wg_t, want_dwg=True))
    for v in ("V1", "V2", "V3"):
        os.environ.pop("HM_UNPERMUTE_" + v, None)
    out["unpermute_router_bwd_ms"] = {v: min(uv[v]) for v in ("v1", "v2", "v3")}
    for v in ("v2", "v3"):
        out[f"unpermute_{v}_bitwise_equal"] = all(
            (a is None and b is None) or bool(torch.equal(a, b)) for a, b in zip(uv["v1_out"], uv[v + "_out"]))
    ub = T * k * d * 2 + T * d * 2
    out["unpermute_router_bwd_gbs"] = {v: ub / ms / 1e6 for v, ms in out["unpermute_router_bwd_ms"].items()}
    a, b = res["tok_dwg"], res["perm_dwg"]
    out["dwg_rel_diff_tok_vs_perm"] = float((a - b).norm() / b.norm())
    fwd_bytes = T * d * 2 + d * E * 2 + T * k * 8 + 8 * E
    bwd_bytes = 2 * T * k * d * 2 + T * d * 2  # unpermute + dlogit.Wg, dWg from x (token-major)
    out["router_fwd_gbs"] = fwd_bytes / out["router_fwd_ms"] / 1e6
    out["router_bwd_gbs"] = {v: bwd_bytes / ms / 1e6 for v, ms in out["router_bwd_ms"].items()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
