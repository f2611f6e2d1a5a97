"""Calibration: our grouped K3 GEMMs vs cuBLAS (torch.bmm) on the same per-expert shapes of the
C2 layer (8 experts x 4096 rows), interleaved so both see the same power/clock state. Prints
TFLOP/s per GEMM and the median SM clock over each measurement."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2504_03871_b200 import _native, ops  # noqa: E402

E, R, d, f = 8, 4096, 4096, 14336
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
rnd = lambda *s: (torch.randn(s, generator=g, device=dev) * 0.05).to(torch.bfloat16)  # noqa: E731
x = rnd(E * R, d)
w_ug = rnd(E, 2 * f, d)
w_d = rnd(E, d, f)
seg = torch.arange(0, E * R + 1, R, dtype=torch.int32, device=dev)
act = rnd(E * R, f)
h = rnd(E * R, 2 * f)
dh = rnd(E * R, 2 * f)
dy = rnd(E * R, d)
out_h = torch.empty(E * R, 2 * f, dtype=torch.bfloat16, device=dev)
out_a = torch.empty(E * R, f, dtype=torch.bfloat16, device=dev)
out_d = torch.empty(E * R, d, dtype=torch.bfloat16, device=dev)
gw_ug = torch.empty(E, 2 * f, d, dtype=torch.bfloat16, device=dev)
gw_d = torch.empty(E, d, f, dtype=torch.bfloat16, device=dev)

ours = {
    "fwd_upgate": (lambda: ops.grouped_gemm(_native.GEMM_FWD_UPGATE, x, w_ug, seg, E, E * R, 0, 2 * f, d, out_a, f,
                                            out2=out_h, ldo2=2 * f), 2 * E * R * d * 2 * f),
    "fwd_down": (lambda: ops.grouped_gemm(_native.GEMM_FWD_DOWN, act, w_d, seg, E, E * R, 0, d, f, out_d, d),
                 2 * E * R * f * d),
    "bwd_dact": (lambda: ops.grouped_gemm(_native.GEMM_BWD_DACT, dy, w_d, seg, E, E * R, 0, f, d, dh, 2 * f,
                                          aux=h, ld_aux=2 * f), 2 * E * R * d * f),
    "bwd_dx": (lambda: ops.grouped_gemm(_native.GEMM_BWD_DX, dh, w_ug, seg, E, E * R, 0, d, 2 * f, out_d, d),
               2 * E * R * 2 * f * d),
    "wgrad_ug": (lambda: ops.grouped_gemm(_native.GEMM_WGRAD, dh, x, seg, E, E * R, 2 * f, d, 0, gw_ug, d),
                 2 * E * R * 2 * f * d),
    "wgrad_down": (lambda: ops.grouped_gemm(_native.GEMM_WGRAD, dy, act, seg, E, E * R, d, f, 0, gw_d, f),
                   2 * E * R * d * f),
}
xb, actb, dyb, dhb = (t.view(E, R, -1) for t in (x, act, dy, dh))
cublas = {
    "fwd_upgate": lambda: torch.bmm(xb, w_ug.transpose(1, 2)),
    "fwd_down": lambda: torch.bmm(actb, w_d.transpose(1, 2)),
    "bwd_dact": lambda: torch.bmm(dyb, w_d),
    "bwd_dx": lambda: torch.bmm(dhb, w_ug),
    "wgrad_ug": lambda: torch.bmm(dhb.transpose(1, 2), xb),
    "wgrad_down": lambda: torch.bmm(dyb.transpose(1, 2), actb),
}


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, clk.summary().get("sm_mhz")


print(f"{'gemm':12s} {'ours TF/s':>10s} {'MHz':>6s} {'cuBLAS TF/s':>12s} {'MHz':>6s} {'ours/cuBLAS per-clock':>22s}")
for name, (fn, flop) in ours.items():
    for _ in range(2):
        t_o, c_o = timeit(fn)
        t_c, c_c = timeit(cublas[name])
    tf_o, tf_c = flop / t_o / 1e9, flop / t_c / 1e9
    pc = (tf_o / c_o) / (tf_c / c_c) if c_o and c_c else float("nan")
    print(f"{name:12s} {tf_o:10.1f} {c_o!s:>6s} {tf_c:12.1f} {c_c!s:>6s} {pc:22.3f}")
