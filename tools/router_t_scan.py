"""Router forward (hm_router_topk, called straight through the C ABI with preallocated outputs)
device time vs token count: the slope is the per-token loop cost, the intercept the prologue /
tail (weight load, last-CTA scan, launch ramp). GPU box only.

    python tools/router_t_scan.py d E k
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_03871_b200 import _native  # noqa: E402


def main():
    d, E, k = (int(v) for v in sys.argv[1:4])
    lib = _native.load()
    dev = torch.device("cuda")
    torch.manual_seed(0)
    busy = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    wg = (torch.randn(d, E, device=dev) * d ** -0.5).bfloat16()
    stream = torch.cuda.current_stream().cuda_stream
    out = {}
    for T in (4096, 8192, 16384, 32768, 65536, 131072):
        x = torch.randn(T, d, device=dev).bfloat16()
        idx = torch.empty((T, k), dtype=torch.int32, device=dev)
        w = torch.empty((T, k), dtype=torch.float32, device=dev)
        logits = torch.empty((T, E), dtype=torch.float32, device=dev)
        counts = torch.empty((E,), dtype=torch.int32, device=dev)
        offsets = torch.empty((E + 1,), dtype=torch.int32, device=dev)
        chunk = torch.empty((max(lib.hm_router_chunk_elems(T, E), 1),), dtype=torch.int32, device=dev)

        def call():
            rc = lib.hm_router_topk(x.data_ptr(), wg.data_ptr(), None, T, d, E, k, idx.data_ptr(), w.data_ptr(),
                                    logits.data_ptr(), counts.data_ptr(), offsets.data_ptr(), chunk.data_ptr(),
                                    stream)
            assert rc == 0

        for _ in range(3):
            call()
        ts = []
        for _ in range(15):
            for _ in range(3):
                busy @ busy
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                call()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 20)
        ts.sort()
        out[T] = round(ts[len(ts) // 2] * 1000, 2)
    print(json.dumps({"d": d, "E": E, "k": k, "us_per_call": out}))


if __name__ == "__main__":
    main()
