"""Per-GEMM cycle accounting on the C2 layer (run with HM_GEMM_STATS=1 on a GPU box)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_layer_tensors  # noqa: E402
from paper_2504_03871_b200 import _native, ops  # noqa: E402
from paper_2504_03871_b200.configs import CONFIGS  # noqa: E402

assert os.environ.get("HM_GEMM_STATS") == "1"
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
x, wg, w_ug, w_down, dy = make_layer_tensors(cfg, 1, torch.device("cuda"))
lib = _native.load()
buf = (ctypes.c_ulonglong * 8)()
r = ops.router_topk(x, wg, cfg.k)
xp, _, row_of = ops.dispatch_permute(x, r)
for rep in range(2):
    lib.hm_gemm_stats(buf)
    y, h, act = ops.grouped_ffn_fwd(xp, r.offsets, w_ug, w_down)
    names = []
    runs = [("fwd", lambda: ops.grouped_ffn_fwd(xp, r.offsets, w_ug, w_down)),
            ("bwd", lambda: ops.grouped_ffn_bwd(y, xp, h, act, r.offsets, w_ug, w_down))]
    for name, fn in runs:
        lib.hm_gemm_stats(buf)
        fn()
        lib.hm_gemm_stats(buf)
        v = list(buf)
        if rep == 1:
            tot = max(v[2], 1)
            print(f"{name}: MMA waits TMA {v[0]/tot:.3f} (of which tile heads {v[6]/max(v[0],1):.2f}), waits TMEM {v[1]/tot:.3f}, producer waits "
                  f"stage {v[3]/max(v[5],1)/ (tot/max(v[5],1)):.3f}; tiles {v[4]}, leader CTAs {v[5]}")
