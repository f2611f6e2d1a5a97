"""Where the end-to-end (host buffers) C2/C3 step spends its time (GPU box): the bench's e2e loop
with host-side issue timing per step and the caching allocator's cudaMalloc / retry counts.

    python tools/e2e_probe.py [C2|C3] [--steps 10]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_layer_tensors  # noqa: E402
from paper_2504_03871_b200.configs import CONFIGS  # noqa: E402
from paper_2504_03871_b200.layer import moe_forward  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C3")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    dev = torch.device("cuda")
    x, wg, w_ug, w_d, dy = make_layer_tensors(cfg, seed=1234, device=dev)
    params = [wg.requires_grad_(), w_ug.requires_grad_(), w_d.requires_grad_()]
    stream = torch.cuda.current_stream()
    x_host = x.detach().cpu().pin_memory()
    dy_host = dy.detach().cpu().pin_memory()
    y_host = [torch.empty(x_host.shape, dtype=x_host.dtype).pin_memory() for _ in range(2)]
    dx_host = [torch.empty(x_host.shape, dtype=x_host.dtype).pin_memory() for _ in range(2)]
    x_dev = [torch.empty_like(x.detach()) for _ in range(2)]
    dy_dev = [torch.empty_like(dy) for _ in range(2)]
    copy_stream, d2h_stream = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]

    def h2d(i):
        b = i & 1
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[b])
            x_dev[b].copy_(x_host, non_blocking=True)
            dy_dev[b].copy_(dy_host, non_blocking=True)
            copied[b].record(copy_stream)

    def step(i, with_copies=True):
        b = i & 1
        if with_copies:
            stream.wait_event(copied[b])
            h2d(i + 1)
        xin = (x_dev[b] if with_copies else x.detach()).detach().requires_grad_()
        for p in params:
            p.grad = None
        y, _ = moe_forward(xin, *params, cfg.k)
        y.backward(dy_dev[b] if with_copies else dy)
        if with_copies:
            consumed[b].record(stream)
            d2h_stream.wait_event(consumed[b])
            with torch.cuda.stream(d2h_stream):
                y.record_stream(d2h_stream)
                xin.grad.record_stream(d2h_stream)
                y_host[b].copy_(y.detach(), non_blocking=True)
                dx_host[b].copy_(xin.grad, non_blocking=True)

    out = {"config": a.config}
    for mode in ("device", "e2e"):
        wc = mode == "e2e"
        for ev in consumed:
            ev.record(stream)
        h2d(0)
        for i in range(3):
            step(i, wc)
        torch.cuda.synchronize()
        st0 = torch.cuda.memory_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        host = []
        e0.record(stream)
        for i in range(3, 3 + a.steps):
            t = time.perf_counter()
            step(i, wc)
            host.append((time.perf_counter() - t) * 1e3)
        stream.wait_stream(d2h_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        st1 = torch.cuda.memory_stats()
        out[mode] = {"gpu_ms_per_step": round(e0.elapsed_time(e1) / a.steps, 3),
                     "host_issue_ms_per_step": [round(v, 2) for v in host],
                     "cudaMalloc": st1["num_device_alloc"] - st0["num_device_alloc"],
                     "cudaFree": st1["num_device_free"] - st0["num_device_free"],
                     "alloc_retries": st1["num_alloc_retries"] - st0["num_alloc_retries"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
