"""One launch each of cuBLAS bmm and K3 (narrow and wide tile) on the C2 down-projection shape
(8 experts x 4096 rows, N=4096, K=14336), for an ncu --set full comparison."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_03871_b200 import _native, ops  # noqa: E402

E, R, d, f = 8, 4096, 4096, 14336
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
act = (torch.randn(E * R, f, generator=g, device=dev) * 0.05).to(torch.bfloat16)
w_d = (torch.randn(E, d, f, generator=g, device=dev) * 0.05).to(torch.bfloat16)
seg = torch.arange(0, E * R + 1, R, dtype=torch.int32, device=dev)
out = torch.empty(E * R, d, dtype=torch.bfloat16, device=dev)
lib = _native.load()
for _ in range(2):
    torch.bmm(act.view(E, R, f), w_d.transpose(1, 2))
    for m in (0x00, 0x3A):
        lib.hm_debug_set_gemm_wide(m)
        ops.grouped_gemm(_native.GEMM_FWD_DOWN, act, w_d, seg, E, E * R, 0, d, f, out, d)
torch.cuda.synchronize()
print("ok")
