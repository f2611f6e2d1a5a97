"""Phase timeline of one fused-router launch (GPU box, needs a library built with
-DHM_ROUTER_TIMELINE, e.g. `make -C paper_2504_03871_b200/csrc OUT=../../abl/rtl.so
EXTRA=-DHM_ROUTER_TIMELINE`): per-CTA globaltimer stamps relative to the earliest CTA entry.

    python tools/router_timeline.py LIB.so [d E k T]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_03871_b200 import _native  # noqa: E402


def main():
    lib = ctypes.CDLL(os.path.abspath(sys.argv[1]))
    d, E, k, T = (int(v) for v in (sys.argv[2:6] if len(sys.argv) > 5 else (4096, 8, 2, 16384)))
    for name in ("hm_router_topk", "hm_router_chunk_elems"):
        res, argt = _native.SIGNATURES[name]
        getattr(lib, name).restype, getattr(lib, name).argtypes = res, argt
    dev = torch.device("cuda")
    torch.manual_seed(0)
    x = torch.randn(T, d, device=dev).bfloat16()
    wg = (torch.randn(d, E, device=dev) * d ** -0.5).bfloat16()
    idx = torch.empty((T, k), dtype=torch.int32, device=dev)
    w = torch.empty((T, k), dtype=torch.float32, device=dev)
    logits = torch.empty((T, E), dtype=torch.float32, device=dev)
    counts = torch.empty((E,), dtype=torch.int32, device=dev)
    offsets = torch.empty((E + 1,), dtype=torch.int32, device=dev)
    chunk = torch.empty((max(lib.hm_router_chunk_elems(T, E), 1),), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    busy = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    res = []
    for rep in range(6):
        busy @ busy
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        rc = lib.hm_router_topk(x.data_ptr(), wg.data_ptr(), None, T, d, E, k, idx.data_ptr(), w.data_ptr(),
                                logits.data_ptr(), counts.data_ptr(), offsets.data_ptr(), chunk.data_ptr(), stream)
        b.record()
        assert rc == 0
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (512 * 5))()
        assert lib.hm_debug_router_timeline(buf) == 0
        tl = [[buf[i * 5 + j] for j in range(5)] for i in range(512)]
        ctas = [r for r in tl[:511] if r[0]]
        t0 = min(r[0] for r in ctas)
        us = lambda v: round((v - t0) / 1e3, 2)  # noqa: E731
        col = lambda j: sorted(us(r[j]) for r in ctas if r[j])  # noqa: E731
        summ = {}
        for j, name in enumerate(("entry", "weights_ready", "compute_done", "epilogue_done", "exit")):
            c = col(j)
            summ[name] = {"min": c[0], "median": c[len(c) // 2], "max": c[-1]}
        summ["scan"] = [us(tl[511][0]), us(tl[511][1])]
        summ["event_ms"] = round(a.elapsed_time(b), 4)
        summ["ctas"] = len(ctas)
        res.append(summ)
    print(json.dumps({"d": d, "E": E, "k": k, "T": T, "runs": res[-3:]}))


if __name__ == "__main__":
    main()
