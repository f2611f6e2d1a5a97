"""Run the C2 per-expert GEMM shapes once through cuBLAS (torch.bmm) and once through K3, for an
ncu capture comparing kernel configurations (tools/gemm_vs_cublas.py has the timing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_03871_b200 import _native, ops  # noqa: E402

E, R, d, f = 8, 4096, 4096, 14336
dev = torch.device("cuda")
rnd = lambda *s: (torch.randn(s, device=dev) * 0.05).to(torch.bfloat16)  # noqa: E731
dh = rnd(E * R, 2 * f)
w_ug = rnd(E, 2 * f, d)
act = rnd(E * R, f)
w_d = rnd(E, d, f)
out_d = torch.empty(E * R, d, dtype=torch.bfloat16, device=dev)
seg = torch.arange(0, E * R + 1, R, dtype=torch.int32, device=dev)
for _ in range(2):
    torch.bmm(act.view(E, R, f), w_d.transpose(1, 2))  # fwd_down
    torch.bmm(dh.view(E, R, 2 * f), w_ug)  # bwd_dx
    ops.grouped_gemm(_native.GEMM_FWD_DOWN, act, w_d, seg, E, E * R, 0, d, f, out_d, d)
    ops.grouped_gemm(_native.GEMM_BWD_DX, dh, w_ug, seg, E, E * R, 0, d, 2 * f, out_d, d)
torch.cuda.synchronize()
