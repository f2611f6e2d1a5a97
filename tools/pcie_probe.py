"""Pinned host<->device copy bandwidth on the GPU box (one direction at a time, then both at once)."""
import torch, time, json
dev = torch.device('cuda')
out = {}
for mib in (64, 256):
    n = mib * 2**20 // 2
    h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    d = torch.empty(n, dtype=torch.bfloat16, device=dev)
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5): fn()
        b.record(); torch.cuda.synchronize()
        out[f"{name}_{mib}MiB_GBps"] = round(5 * mib * 2**20 / (a.elapsed_time(b) / 1e3) / 1e9, 1)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h2 = torch.empty(n, dtype=torch.bfloat16).pin_memory(); d2 = torch.empty_like(d)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); out[f"bidir_{mib}MiB_GBps_each"] = round(5 * mib * 2**20 / (time.perf_counter() - t) / 1e9, 1)
print(json.dumps(out))
