"""Same-process A/B of two builds of libhetermoe_kernels.so on the router forward (K1,
hm_router_topk) of one config (GPU box only): both libraries are loaded side by side with ctypes
and timed alternately A, B, A, B, ... (CUDA events over `--inner` back-to-back calls, each batch
queued behind a matmul so host launch latency never starves the GPU; median of --reps rounds).
Also checks that both builds produce the same bits.

    python tools/ab_router.py OLD.so NEW.so [--config C2] [--reps 15]
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_layer_tensors  # noqa: E402
from paper_2504_03871_b200 import _native  # noqa: E402
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
    x, wg, _, _, _ = make_layer_tensors(cfg, 1, dev)
    T, d = x.shape
    E, k = wg.shape[1], cfg.k
    libs, outs = [], []
    for p in (args.lib_a, args.lib_b):
        lib = ctypes.CDLL(os.path.abspath(p))
        for name in ("hm_router_topk", "hm_router_chunk_elems"):
            res, argt = _native.SIGNATURES[name]
            getattr(lib, name).restype, getattr(lib, name).argtypes = res, argt
        nce = max(lib.hm_router_chunk_elems(T, E), 1)
        o = dict(idx=torch.empty((T, k), dtype=torch.int32, device=dev),
                 w=torch.empty((T, k), dtype=torch.float32, device=dev),
                 logits=torch.empty((T, E), dtype=torch.float32, device=dev),
                 counts=torch.empty((E,), dtype=torch.int32, device=dev),
                 offsets=torch.empty((E + 1,), dtype=torch.int32, device=dev),
                 chunk=torch.empty((nce,), dtype=torch.int32, device=dev))
        libs.append(lib)
        outs.append(o)
    stream = torch.cuda.current_stream().cuda_stream

    def call(i):
        o = outs[i]
        rc = libs[i].hm_router_topk(x.data_ptr(), wg.data_ptr(), None, T, d, E, k, o["idx"].data_ptr(),
                                    o["w"].data_ptr(), o["logits"].data_ptr(), o["counts"].data_ptr(),
                                    o["offsets"].data_ptr(), o["chunk"].data_ptr(), stream)
        assert rc == 0, rc

    busy = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    for i in (0, 1):
        for _ in range(3):
            call(i)
    torch.cuda.synchronize()
    same = {n: bool(torch.equal(outs[0][n], outs[1][n])) for n in ("idx", "w", "logits", "counts", "offsets")}
    ts = [[], []]
    for _ in range(args.reps):
        for i in (0, 1):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            for _ in range(3):
                busy @ busy
            a.record()
            for _ in range(args.inner):
                call(i)
            b.record()
            torch.cuda.synchronize()
            ts[i].append(a.elapsed_time(b) / args.inner)
    med = [sorted(t)[len(t) // 2] for t in ts]
    print(json.dumps({"config": args.config, "a": args.lib_a, "b": args.lib_b, "bitwise_equal": same,
                      "ms_med": {"a": round(med[0], 5), "b": round(med[1], 5)},
                      "ms_best": {"a": round(min(ts[0]), 5), "b": round(min(ts[1]), 5)}}))


if __name__ == "__main__":
    main()
