"""K2 dispatch-permute timing with 1, 2, 4 CTAs per 64-token chunk (HM_PERMUTE_SPLIT), outputs
compared bitwise against split 1 (GPU box).

    python tools/permute_bench.py [C2|C3] [--reps 20]
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
from tools.router_bench import timed  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C3")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    x, wg, *_ = make_layer_tensors(cfg, 1, torch.device("cuda"))
    r = ops.router_topk(x, wg, cfg.k)
    out = {"config": args.config, "ms": {}, "bitwise_equal": {}}
    ref = None
    for split in (1, 2, 4, 8, 1, 2, 4, 8):
        os.environ["HM_PERMUTE_SPLIT"] = str(split)
        ms = timed(lambda: ops.dispatch_permute(x, r), args.reps)
        out["ms"][split] = min(ms, out["ms"].get(split, 1e9))
        res = ops.dispatch_permute(x, r)
        if ref is None:
            ref = res
        out["bitwise_equal"][split] = all(bool(torch.equal(a, b)) for a, b in zip(ref, res))
    os.environ.pop("HM_PERMUTE_SPLIT", None)
    nbytes = cfg.T * cfg.d * 2 * (1 + cfg.k)
    out["gbs"] = {s: nbytes / ms / 1e6 for s, ms in out["ms"].items()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
