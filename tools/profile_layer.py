"""Run a few C2 (or --config) MoE-layer fwd+bwd steps for ncu captures (no timing printed)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_layer_tensors  # noqa: E402
from paper_2504_03871_b200.configs import CONFIGS, with_tokens  # noqa: E402
from paper_2504_03871_b200.layer import moe_forward  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--tokens", type=int, default=0)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
cfg = CONFIGS[a.config] if not a.tokens else with_tokens(CONFIGS[a.config], a.tokens)
x, wg, w_ug, w_down, dy = make_layer_tensors(cfg, 1, torch.device("cuda"))
ps = [wg.requires_grad_(), w_ug.requires_grad_(), w_down.requires_grad_()]
x.requires_grad_()
for _ in range(a.steps):
    for p in ps + [x]:
        p.grad = None
    y, _ = moe_forward(x, *ps, cfg.k)
    y.backward(dy)
torch.cuda.synchronize()
print("ok")
