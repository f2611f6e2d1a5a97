"""A/B of K3 launch configurations on the full C2 layer step (GPU box): blocks of --block steps
alternate between the variants in ONE process, so clock / power drift hits all alike; prints the
median ms per step of each variant.

    python tools/ab_step.py [--config C2] [--rounds 6] [--block 4]
Variants: "r2" = the library defaults; "r1" = round-1 launch choices (narrow SwiGLU backward,
raster group height 8 for every GEMM)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_layer_tensors  # noqa: E402
from paper_2504_03871_b200 import _native  # noqa: E402
from paper_2504_03871_b200.configs import CONFIGS  # noqa: E402
from paper_2504_03871_b200.layer import moe_forward  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--block", type=int, default=4)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    lib = _native.load()
    x, wg, w_ug, w_d, dy = make_layer_tensors(cfg, 1, torch.device("cuda"))
    ps = [wg.requires_grad_(), w_ug.requires_grad_(), w_d.requires_grad_()]
    x.requires_grad_()

    def select(v):
        if v == "r1":
            lib.hm_debug_set_gemm_wide(0x3B)
            lib.hm_debug_set_gemm_groupm(-1, 8)
        else:
            lib.hm_debug_set_gemm_wide(-1)
            lib.hm_debug_set_gemm_groupm(-1, 0)

    def block():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.block):
            for p in ps + [x]:
                p.grad = None
            y, _ = moe_forward(x, *ps, cfg.k)
            y.backward(dy)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.block

    variants = ["r1", "r2"]
    for v in variants:
        select(v)
        block()
    res = {v: [] for v in variants}
    for _ in range(args.rounds):
        for v in variants:
            select(v)
            res[v].append(block())
    out = {v: {"ms_med": sorted(t)[len(t) // 2], "ms_all": [round(q, 3) for q in t]} for v, t in res.items()}
    out["tokens_per_s_med"] = {v: cfg.T / (out[v]["ms_med"] / 1e3) for v in variants}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
