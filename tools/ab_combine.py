"""Same-process A/B of two builds of libhetermoe_kernels.so on K4 (hm_combine, hm_combine_bwd)
and K2 (hm_dispatch_permute) for one config (GPU box): alternating batches of back-to-back calls
(CUDA events, median of --reps), outputs compared bitwise.

    python tools/ab_combine.py OLD.so NEW.so [--config C2] [--reps 15]
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
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--inner", type=int, default=10)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    dev = torch.device("cuda")
    x, wg, _, _, dy = make_layer_tensors(cfg, 1, dev)
    r = ops.router_topk(x, wg, cfg.k)
    xp, _, row_of = ops.dispatch_permute(x, r)
    T, d, k, E = cfg.T, cfg.d, cfg.k, cfg.E
    libs = []
    for p in (args.lib_a, args.lib_b):
        lib = ctypes.CDLL(os.path.abspath(p))
        for n in ("hm_combine", "hm_combine_bwd", "hm_dispatch_permute"):
            res, argt = _native.SIGNATURES[n]
            getattr(lib, n).restype, getattr(lib, n).argtypes = res, argt
        libs.append(lib)
    st = torch.cuda.current_stream().cuda_stream
    outs = [dict(y=torch.empty((T, d), dtype=torch.bfloat16, device=dev),
                 dyp=torch.empty_like(xp), dw=torch.empty((T, k), dtype=torch.float32, device=dev),
                 xp=torch.empty_like(xp), rs=torch.empty((T * k,), dtype=torch.int32, device=dev),
                 ro=torch.empty((T, k), dtype=torch.int32, device=dev)) for _ in libs]
    P = lambda t: t.data_ptr()  # noqa: E731
    calls = {
        "combine": lambda i: libs[i].hm_combine(P(xp), P(row_of), P(r.w), T, d, k, P(outs[i]["y"]), st),
        "combine_bwd": lambda i: libs[i].hm_combine_bwd(P(dy), P(xp), P(row_of), P(r.w), T, d, k,
                                                        P(outs[i]["dyp"]), P(outs[i]["dw"]), st),
        "dispatch_permute": lambda i: libs[i].hm_dispatch_permute(P(x), P(r.idx), P(r.chunk_base), T, d, E, k,
                                                                  P(outs[i]["xp"]), P(outs[i]["rs"]),
                                                                  P(outs[i]["ro"]), st),
    }
    busy = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    res = {"config": args.config}
    for name, fn in calls.items():
        for i in (0, 1):
            assert fn(i) == 0
        torch.cuda.synchronize()
        ts = [[], []]
        for _ in range(args.reps):
            for i in (0, 1):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                for _ in range(3):
                    busy @ busy
                a.record()
                for _ in range(args.inner):
                    fn(i)
                b.record()
                torch.cuda.synchronize()
                ts[i].append(a.elapsed_time(b) / args.inner)
        med = [sorted(t)[len(t) // 2] for t in ts]
        res[name] = {"ms_a": round(med[0], 5), "ms_b": round(med[1], 5)}
    res["bitwise_equal"] = {n: all(torch.equal(outs[0][n], outs[1][n]) for _ in [0]) for n in outs[0]}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
