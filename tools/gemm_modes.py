"""Per-GEMM timing (and, with HM_GEMM_STATS=1, cycle accounting) of the six K3 launches of the
C2 layer, each run alone back to back (CUDA events, median of --reps). GPU box only.

    python tools/gemm_modes.py [C2|C3] [--reps 20]
Environment knobs read by the library (HM_GEMM_WIDE, HM_GEMM_GROUPM, HM_GEMM_STATS) select variants;
run one process per setting."""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_layer_tensors  # noqa: E402
from paper_2504_03871_b200 import _native, ops  # noqa: E402
from paper_2504_03871_b200.configs import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ab", default="", help="comma-separated variants 'WIDE_MASK[:GROUP_M]' timed "
                    "interleaved (e.g. 0x3A:8,0x3A:16)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    dev = torch.device("cuda")
    x, wg, w_ug, w_d, dy = make_layer_tensors(cfg, 1, dev)
    lib = _native.load()
    stats = os.environ.get("HM_GEMM_STATS") == "1"
    buf = (ctypes.c_ulonglong * 8)()
    r = ops.router_topk(x, wg, cfg.k)
    xp, _, row_of = ops.dispatch_permute(x, r)
    rows, d = xp.shape
    E, two_f, _ = w_ug.shape
    f = two_f // 2
    seg = r.offsets
    y, h, act = ops.grouped_ffn_fwd(xp, seg, w_ug, w_d)
    dyp = torch.randn_like(y)
    dh = torch.empty((rows, 2 * f), dtype=xp.dtype, device=dev)
    dxp = torch.empty((rows, d), dtype=xp.dtype, device=dev)
    dw_ug = torch.empty_like(w_ug)
    dw_d = torch.empty_like(w_d)
    G = _native
    gemms = {
        "fwd_upgate": (lambda: ops.grouped_gemm(G.GEMM_FWD_UPGATE, xp, w_ug, seg, E, rows, 0, 2 * f, d, act, f,
                                                out2=h, ldo2=2 * f), 2 * rows * d * 2 * f),
        "fwd_down": (lambda: ops.grouped_gemm(G.GEMM_FWD_DOWN, act, w_d, seg, E, rows, 0, d, f, y, d),
                     2 * rows * f * d),
        "bwd_dact": (lambda: ops.grouped_gemm(G.GEMM_BWD_DACT, dyp, w_d, seg, E, rows, 0, f, d, dh, 2 * f,
                                              aux=h, ld_aux=2 * f), 2 * rows * d * f),
        "bwd_dx": (lambda: ops.grouped_gemm(G.GEMM_BWD_DX, dh, w_ug, seg, E, rows, 0, d, 2 * f, dxp, d),
                   2 * rows * 2 * f * d),
        "wgrad_ug": (lambda: ops.grouped_gemm(G.GEMM_WGRAD, dh, xp, seg, E, rows, 2 * f, d, 0, dw_ug, d),
                     2 * rows * 2 * f * d),
        "wgrad_down": (lambda: ops.grouped_gemm(G.GEMM_WGRAD, dyp, act, seg, E, rows, d, f, 0, dw_d, f),
                       2 * rows * d * f),
    }
    out = {"config": args.config, "env": {k: v for k, v in os.environ.items() if k.startswith("HM_")}}
    masks = args.ab.split(",") if args.ab else [None]

    def select(m):
        # WIDE_MASK[:GROUP_M[:EARLY_RELEASE]]
        parts = m.split(":")
        lib.hm_debug_set_gemm_wide(int(parts[0], 0))
        lib.hm_debug_set_gemm_groupm(-1, int(parts[1]) if len(parts) > 1 and parts[1] else 0)
        lib.hm_debug_set_gemm_early_release(int(parts[2]) if len(parts) > 2 else 1)

    def one(fn):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    for name, (fn, flops) in gemms.items():
        for m in masks:
            if m is not None:
                select(m)
            for _ in range(2):
                fn()
        torch.cuda.synchronize()
        ts = {m: [] for m in masks}
        for _ in range(args.reps):  # variants interleaved so clock / power drift hits all alike
            for m in masks:
                if m is not None:
                    select(m)
                ts[m].append(one(fn))
        for m in masks:
            t = sorted(ts[m])
            med = t[len(t) // 2]
            rec = {"ms_med": round(med, 4), "ms_best": round(t[0], 4),
                   "tflops_med": round(flops / med / 1e9, 1)}
            if stats:
                if m is not None:
                    select(m)
                lib.hm_gemm_stats(buf)
                fn()
                lib.hm_gemm_stats(buf)
                v = list(buf)
                tot = max(v[2], 1)
                rec["mma_wait_tma"] = round(v[0] / tot, 3)
                rec["mma_wait_tmem"] = round(v[1] / tot, 3)
                rec["head_share_of_tma_wait"] = round(v[6] / max(v[0], 1), 3)
                rec["producer_wait_stage"] = round(v[3] / tot, 3)
                rec["tiles"] = v[4]
            out[name if m is None else f"{name}@{m}"] = rec
        if masks[0] is not None:
            lib.hm_debug_set_gemm_wide(-1)
            lib.hm_debug_set_gemm_groupm(-1, 0)
            lib.hm_debug_set_gemm_early_release(1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
