"""Same-process A/B of two builds of libhetermoe_kernels.so on the six K3 GEMMs of one layer
config (GPU box only): both libraries are loaded side by side with ctypes and every GEMM is timed
alternately A, B, A, B, ... (CUDA events, median of --reps rounds), so clock / power drift hits
both builds alike.

    python tools/ab_libs.py OLD.so NEW.so [--config C2] [--reps 9]
"""
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
    ap.add_argument("lib_a")
    ap.add_argument("lib_b")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=9)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    dev = torch.device("cuda")
    libs = []
    for p in (args.lib_a, args.lib_b):
        lib = ctypes.CDLL(os.path.abspath(p))
        res, argt = _native.SIGNATURES["hm_grouped_gemm"]
        lib.hm_grouped_gemm.restype, lib.hm_grouped_gemm.argtypes = res, argt
        lib.hm_grouped_gemm_workspace_bytes.restype = ctypes.c_size_t
        libs.append(lib)
    x, wg, w_ug, w_d, dy = make_layer_tensors(cfg, 1, dev)
    r = ops.router_topk(x, wg, cfg.k)
    xp, _, _ = ops.dispatch_permute(x, r)
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
    ws = torch.empty((4096,), dtype=torch.uint8, device=dev)
    wsp = ws.data_ptr() + (-ws.data_ptr()) % 128
    P = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    G = _native
    # (mode, a, b, M, N, K, out, ldo, out2, ldo2, aux, ld_aux, flops)
    gemms = {
        "fwd_upgate": (G.GEMM_FWD_UPGATE, xp, w_ug, 0, 2 * f, d, act, f, h, 2 * f, None, 0, 2 * rows * d * 2 * f),
        "fwd_down": (G.GEMM_FWD_DOWN, act, w_d, 0, d, f, y, d, None, 0, None, 0, 2 * rows * f * d),
        "bwd_dact": (G.GEMM_BWD_DACT, dyp, w_d, 0, f, d, dh, 2 * f, None, 0, h, 2 * f, 2 * rows * d * f),
        "bwd_dx": (G.GEMM_BWD_DX, dh, w_ug, 0, d, 2 * f, dxp, d, None, 0, None, 0, 2 * rows * 2 * f * d),
        "wgrad_ug": (G.GEMM_WGRAD, dh, xp, 2 * f, d, 0, dw_ug, d, None, 0, None, 0, 2 * rows * 2 * f * d),
        "wgrad_down": (G.GEMM_WGRAD, dyp, act, d, f, 0, dw_d, f, None, 0, None, 0, 2 * rows * d * f),
    }
    stream = torch.cuda.current_stream().cuda_stream

    def call(lib, g):
        mode, a, b, M, N, K, out, ldo, out2, ldo2, aux, ld_aux, _ = g
        rc = lib.hm_grouped_gemm(mode, P(a), P(b), P(seg), E, rows, M, N, K, P(out), ldo, P(out2), ldo2, P(aux),
                                 ld_aux, wsp, 0, stream)
        assert rc == 0, rc

    res = {}
    for name, g in gemms.items():
        for lib in libs:  # warm-up
            call(lib, g)
        ts = [[], []]
        for _ in range(args.reps):
            for i, lib in enumerate(libs):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(3):
                    call(lib, g)
                e1.record()
                torch.cuda.synchronize()
                ts[i].append(e0.elapsed_time(e1) / 3)
        med = [sorted(t)[len(t) // 2] for t in ts]
        res[name] = {"a_ms": round(med[0], 4), "b_ms": round(med[1], 4), "b_over_a": round(med[1] / med[0], 4),
                     "a_tflops": round(g[-1] / med[0] / 1e9, 1), "b_tflops": round(g[-1] / med[1] / 1e9, 1)}
    tot = [sum(v["a_ms"] for v in res.values()), sum(v["b_ms"] for v in res.values())]
    print(json.dumps({"config": args.config, "a": args.lib_a, "b": args.lib_b, "gemms": res,
                      "total_ms": [round(t, 3) for t in tot], "b_over_a": round(tot[1] / tot[0], 4)}))


if __name__ == "__main__":
    main()
