"""Router backward timed INSIDE the C2 layer step (the bench's per-op CUDA events), alternating the
one-pass kernel (HM_ROUTER_BWD_FUSED) and the default two-pass path in one process. GPU box only."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_layer_tensors  # noqa: E402
from paper_2504_03871_b200 import ops  # noqa: E402
from paper_2504_03871_b200.configs import CONFIGS  # noqa: E402
from paper_2504_03871_b200.layer import moe_forward  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
x, wg, w_ug, w_d, dy = make_layer_tensors(cfg, 1, torch.device("cuda"))
ps = [wg.requires_grad_(), w_ug.requires_grad_(), w_d.requires_grad_()]
x.requires_grad_()
res = {}
for rnd in range(6):
    for v in ("fused", "two_pass"):
        if v == "fused":
            os.environ["HM_ROUTER_BWD_FUSED"] = "1"
        else:
            os.environ.pop("HM_ROUTER_BWD_FUSED", None)
        timer = ops.KernelTimer()
        ops.set_timer(timer)
        for _ in range(3):
            for p in ps + [x]:
                p.grad = None
            y, _ = moe_forward(x, *ps, cfg.k)
            y.backward(dy)
        torch.cuda.synchronize()
        ops.set_timer(None)
        if rnd:
            summ = timer.summary()
            res.setdefault(v, []).append(summ["router_bwd"][1] / summ["router_bwd"][0])
os.environ.pop("HM_ROUTER_BWD_FUSED", None)
print(json.dumps({v: {"ms_med": sorted(t)[len(t) // 2], "all": [round(q, 4) for q in t]} for v, t in res.items()}))
