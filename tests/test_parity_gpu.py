"""GPU parity against the CPU oracle at the BASELINE layer shapes and on adversarial routing rows
(run on a B200). Complements test_kernels_gpu.py.

Bars, written here as in the sibling file: routing indices, counts, offsets, row
maps and permuted rows BIT-EXACT; gate weights within 1e-5 abs (NaN where the oracle has NaN);
layer output and dX within relative Frobenius error 1e-2 of the fp32 oracle fed the same bf16
inputs; weight gradients within 2e-2.
"""

import numpy as np
import pytest
import torch

from oracle import moe_oracle as orc
from paper_2504_03871_b200 import ops
from paper_2504_03871_b200.configs import C2, C3, LayerConfig, make_inputs, with_tokens

pytestmark = pytest.mark.gpu

TOL_ACT = 1e-2
TOL_W = 2e-2
TOL_GATE = 1e-5


def _same_float(a: np.ndarray, b: np.ndarray) -> bool:
    """Bitwise equal where finite or infinite; NaN where the other is NaN (payloads may differ)."""
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    return np.array_equal(a[~na].view(np.uint32), b[~nb].view(np.uint32))


# one config per top-k kernel: fused logits+top-k (E=8, E=16), thread-per-token (E=64, C3 shape),
# warp-per-token (E=256); T not a multiple of the 64-token chunk
ADV_CASES = [
    LayerConfig("E8k2", E=8, k=2, d=4096, f=128, T=203),
    LayerConfig("E16k4", E=16, k=4, d=512, f=128, T=130),
    LayerConfig("E64k6", E=64, k=6, d=2048, f=128, T=257),
    LayerConfig("E256k8", E=256, k=8, d=256, f=128, T=99),
    LayerConfig("E8k8", E=8, k=8, d=256, f=128, T=65),
]


def _adversarial_x(x: torch.Tensor) -> torch.Tensor:
    x = x.clone()
    x[1] = 0  # all logits 0 (+ bias): an all-tie row
    x[2] = float("nan")  # all-NaN row
    x[3] = 0
    x[3, 5] = float("inf")  # +inf / -inf logits by the sign of Wg[5, e]
    x[4, 7] = float("nan")  # NaN in one element -> all-NaN logits too
    x[5] = 0
    x[5, 0] = float("-inf")
    x[-1] = 0  # last (ragged) chunk gets a tie row
    return x


def _bias_variants(E):
    nan_free = np.zeros(E, dtype=np.float32)
    half_ninf = np.zeros(E, dtype=np.float32)
    half_ninf[1::2] = -np.inf  # more -inf experts than k -> -inf ties must still pick distinct ids
    one_left = np.full(E, -np.inf, dtype=np.float32)
    one_left[E - 1] = 0.0  # only the last expert finite
    return {"none": None, "zero": nan_free, "half_-inf": half_ninf, "one_finite": one_left}


@pytest.mark.parametrize("bias_name", ["none", "zero", "half_-inf", "one_finite"])
@pytest.mark.parametrize("cfg", ADV_CASES, ids=lambda c: c.name)
def test_router_nonfinite_and_tie_rows_vs_oracle(cfg, bias_name):
    inp = make_inputs(cfg, seed=13)
    x = _adversarial_x(inp.x)
    bias = _bias_variants(cfg.E)[bias_name]
    ref = orc.route(x.float().numpy(), inp.wg.float().numpy(), cfg.k, bias=bias)
    xc = x.cuda()
    r = ops.router_topk(xc, inp.wg.cuda(), cfg.k, None if bias is None else torch.from_numpy(bias).cuda())
    x_perm, row_src, row_of = ops.dispatch_permute(xc, r)
    torch.cuda.synchronize()
    assert _same_float(r.logits.cpu().numpy(), ref.logits), "logits"
    idx = r.idx.cpu().numpy()
    assert np.array_equal(idx, ref.idx), np.nonzero((idx != ref.idx).any(1))
    for row in idx:
        assert len(set(row.tolist())) == cfg.k  # never the same expert twice
    np.testing.assert_allclose(r.w.cpu().numpy(), ref.w, rtol=0, atol=TOL_GATE)  # NaN == NaN
    assert np.array_equal(r.counts.cpu().numpy(), ref.counts)
    assert np.array_equal(r.offsets.cpu().numpy(), ref.offsets)
    assert int(r.offsets[-1]) == cfg.T * cfg.k
    assert np.array_equal(row_src.cpu().numpy(), ref.row_src)
    assert np.array_equal(row_of.cpu().numpy(), ref.row_of)
    got = x_perm.cpu().view(torch.int16)
    want = x[torch.from_numpy(ref.row_src.astype(np.int64))].view(torch.int16)
    assert torch.equal(got, want)  # bitwise, NaN/inf rows included


def _layer_vs_oracle(cfg, seed, expert_bias=None, check_empty=None):
    from paper_2504_03871_b200.layer import moe_forward

    inp = make_inputs(cfg, seed=seed, expert_bias=expert_bias)
    w_ug = ops.interleave_gate_up(inp.w_gate, inp.w_up)
    x = inp.x.cuda().requires_grad_()
    wg = inp.wg.cuda().requires_grad_()
    wug = w_ug.cuda().requires_grad_()
    wd = inp.w_down.cuda().requires_grad_()
    y, idx = moe_forward(x, wg, wug, wd, cfg.k)
    y.backward(inp.dy.cuda())
    torch.cuda.synchronize()
    got = {"y": y.cpu(), "dx": x.grad.cpu(), "dwg": wg.grad.cpu(), "dw_down": wd.grad.cpu()}
    got["dw_gate"], got["dw_up"] = ops.split_gate_up(wug.grad.cpu())
    idx = idx.cpu().numpy()
    del x, wg, wug, wd, y
    torch.cuda.empty_cache()
    ref = orc.moe_layer(inp.x, inp.wg, w_ug, inp.w_down, cfg.k, dy=inp.dy)
    assert np.array_equal(idx, ref["routing"].idx)
    errs = {
        "y": orc.rel_err(got["y"], ref["y"]),
        "dx": orc.rel_err(got["dx"], ref["dx"]),
        "dwg": orc.rel_err(got["dwg"], ref["dwg"]),
        "dw_gate": orc.rel_err(got["dw_gate"], ref["dw_gate"]),
        "dw_up": orc.rel_err(got["dw_up"], ref["dw_up"]),
        "dw_down": orc.rel_err(got["dw_down"], ref["dw_down"]),
    }
    tol = {"y": TOL_ACT, "dx": TOL_ACT}
    bad = {k: v for k, v in errs.items() if not v < tol.get(k, TOL_W)}
    assert not bad, (bad, errs)
    if check_empty is not None:
        counts = ref["routing"].counts
        assert counts[check_empty] == 0
        assert torch.count_nonzero(got["dw_gate"][check_empty]) == 0
        assert torch.count_nonzero(got["dw_down"][check_empty]) == 0
    return errs


def test_moe_layer_c3_shape_vs_oracle():
    """C3 (E=64, top-6, d=2048, f=1408: partial N tiles in the wide GEMMs, 64 ragged experts)."""
    _layer_vs_oracle(with_tokens(C3, 2048), seed=31)


def test_moe_layer_c2_shape_vs_oracle():
    """C2 (E=8, top-2, d=4096, f=14336): the Mixtral layer at T=2048."""
    _layer_vs_oracle(with_tokens(C2, 2048), seed=32)


def test_moe_layer_with_empty_expert_vs_oracle():
    """An expert that receives no token (router bias -30): zero rows in K3's variable-K weight
    gradient, an empty segment in every GEMM, zero gradient rows for that expert."""
    cfg = LayerConfig("empty-expert", E=8, k=2, d=512, f=384, T=1000)
    bias = [0.0] * 8
    bias[3] = -30.0
    _layer_vs_oracle(cfg, seed=33, expert_bias=bias, check_empty=3)


@pytest.mark.parametrize("cfg", [LayerConfig("E8d4096", 8, 2, 4096, 128, 1000),
                                 LayerConfig("E4d256", 4, 3, 256, 128, 777),
                                 LayerConfig("E8d8192", 8, 2, 8192, 128, 300),
                                 LayerConfig("E2d16384", 2, 1, 16384, 128, 130),
                                 LayerConfig("E8d768", 8, 2, 768, 128, 500),
                                 LayerConfig("E8d1280", 8, 3, 1280, 128, 333),
                                 LayerConfig("E8d6144", 8, 2, 6144, 128, 257),
                                 LayerConfig("E16d7168", 16, 4, 7168, 128, 130),
                                 LayerConfig("E4d12288", 4, 2, 12288, 128, 71)],
                         ids=lambda c: c.name)
def test_router_fused_equals_unfused_and_oracle(cfg):
    """The one-kernel router (logits + top-k + histogram + last-CTA scan, one expert group) and
    the unfused path (logits kernel, top-k kernel, scan kernel; HM_ROUTER_UNFUSED) agree bitwise,
    and both match the oracle, on adversarial rows too; d = 8192 / 16384 exercise the 4- and
    2-expert register groups, d = 768, 1280, 6144 (Mixtral-8x22B), 7168 (DeepSeek-V3), 12288 the
    run-time block count (1, 2 and 3 blocks per warp, idle warps when 16 % (d / 256) != 0)."""
    import os

    inp = make_inputs(cfg, seed=17)
    x = _adversarial_x(inp.x).cuda()
    wg = inp.wg.cuda()
    a = ops.router_topk(x, wg, cfg.k)
    os.environ["HM_ROUTER_UNFUSED"] = "1"
    try:
        b = ops.router_topk(x, wg, cfg.k)
    finally:
        os.environ.pop("HM_ROUTER_UNFUSED")
    torch.cuda.synchronize()
    n = ((cfg.T + 63) // 64) * cfg.E
    for name in ("idx", "counts", "offsets"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    assert torch.equal(a.chunk_base[:n], b.chunk_base[:n])
    assert _same_float(a.logits.cpu().numpy(), b.logits.cpu().numpy())
    assert _same_float(a.w.cpu().numpy(), b.w.cpu().numpy())
    ref = orc.route(x.cpu().float().numpy(), inp.wg.float().numpy(), cfg.k)
    assert _same_float(a.logits.cpu().numpy(), ref.logits)
    assert np.array_equal(a.idx.cpu().numpy(), ref.idx)
    assert np.array_equal(a.offsets.cpu().numpy(), ref.offsets)
    np.testing.assert_allclose(a.w.cpu().numpy(), ref.w, rtol=0, atol=TOL_GATE)


@pytest.mark.parametrize("cfg", [LayerConfig("E8d4096", 8, 2, 4096, 128, 3000),
                                 LayerConfig("E4d1024k3", 4, 3, 1024, 128, 777)], ids=lambda c: c.name)
def test_router_bwd_streamed_wgrad_vs_fp32(cfg):
    """The one-pass router backward (E <= 8, k <= 3: dx and dWg per column tile from the token rows
    and routed dX rows streamed through shared memory), the two-pass streamed dWg, the token-major
    and the per-expert paths: dx and dlogit bitwise equal, dWg against a plain fp32 reference
    x^T . dlogit_dense."""
    import os

    inp = make_inputs(cfg, seed=19)
    x, wg = inp.x.cuda(), inp.wg.cuda()
    r = ops.router_topk(x, wg, cfg.k)
    xp, _, row_of = ops.dispatch_permute(x, r)
    g = torch.Generator(device="cuda").manual_seed(4)
    dxp = torch.randn(xp.shape, generator=g, device="cuda").to(xp.dtype)
    dw = torch.randn(r.w.shape, generator=g, device="cuda")
    wg_t = ops.transpose_bf16(wg)
    outs = {}
    for v, env in (("fused", "HM_ROUTER_BWD_FUSED"), ("stream", None), ("tok", "HM_ROUTER_WGRAD_TOK"),
                   ("perm", "HM_ROUTER_WGRAD_PERM")):
        if env:
            os.environ[env] = "1"
        try:
            outs[v] = ops.router_bwd(dxp, row_of, r, dw, xp, wg_t, want_dwg=True, x=x)
        finally:
            if env:
                os.environ.pop(env)
    torch.cuda.synchronize()
    dl = outs["fused"][1].float()  # dlogit [T, k]
    dense = torch.zeros((cfg.T, cfg.E), device="cuda").scatter_(1, r.idx.long(), dl)
    ref = x.float().t() @ dense
    for v in outs:
        assert torch.equal(outs[v][0], outs["fused"][0]), v  # dx identical on every path
        assert torch.equal(outs[v][1], outs["fused"][1]), v  # dlogit too
        assert orc.rel_err(outs[v][2], ref) < 5e-3, v


@pytest.mark.parametrize("cfg", [LayerConfig("E64d2048k6", 64, 6, 2048, 128, 3000),
                                 LayerConfig("E16d1024k4", 16, 4, 1024, 128, 777)], ids=lambda c: c.name)
def test_router_bwd_gemm_wgrad_vs_fp32(cfg):
    """E > 8: the router weight gradient as a K-split tensor-core GEMM over the token rows (dense
    bf16 dlogit rows, fp32 split partials) against the per-expert path over the routed copies
    (HM_ROUTER_WGRAD_PERM) and a plain fp32 x^T . dlogit_dense; dx and dlogit bitwise equal."""
    import os

    inp = make_inputs(cfg, seed=23)
    x, wg = inp.x.cuda(), inp.wg.cuda()
    r = ops.router_topk(x, wg, cfg.k)
    xp, _, row_of = ops.dispatch_permute(x, r)
    g = torch.Generator(device="cuda").manual_seed(6)
    dxp = torch.randn(xp.shape, generator=g, device="cuda").to(xp.dtype)
    dw = torch.randn(r.w.shape, generator=g, device="cuda")
    wg_t = ops.transpose_bf16(wg)
    gemm = ops.router_bwd(dxp, row_of, r, dw, xp, wg_t, want_dwg=True, x=x)
    os.environ["HM_ROUTER_WGRAD_PERM"] = "1"
    try:
        perm = ops.router_bwd(dxp, row_of, r, dw, xp, wg_t, want_dwg=True, x=x)
    finally:
        os.environ.pop("HM_ROUTER_WGRAD_PERM")
    torch.cuda.synchronize()
    assert torch.equal(gemm[0], perm[0]) and torch.equal(gemm[1], perm[1])
    dense = torch.zeros((cfg.T, cfg.E), device="cuda").scatter_(1, r.idx.long(), gemm[1].float())
    ref = x.float().t() @ dense
    assert orc.rel_err(perm[2], ref) < 5e-3
    assert orc.rel_err(gemm[2], ref) < 5e-3


def test_c_abi_grouped_ffn_entry_points_match_ops():
    """hm_grouped_ffn_fwd / hm_grouped_ffn_bwd — the C-ABI compositions a C/C++ runtime calls for
    EXP_F / EXP_B (include/hetermoe.h) — called through ctypes exactly as INTEGRATION.md shows,
    bitwise equal to the per-GEMM path the Python layer uses, and within the fp32 bars."""
    from paper_2504_03871_b200 import _native

    lib = _native.load()
    segs = [700, 0, 1200, 333, 64, 1]
    E, d, f = len(segs), 512, 384
    rows = sum(segs)
    g = torch.Generator(device="cuda").manual_seed(6)
    bf = lambda *s, std=1.0: (torch.randn(s, generator=g, device="cuda") * std).to(torch.bfloat16)  # noqa: E731
    x, dy = bf(rows, d), bf(rows, d)
    w_ug, w_d = bf(E, 2 * f, d, std=d ** -0.5), bf(E, d, f, std=f ** -0.5)
    off = np.zeros(E + 1, dtype=np.int32)
    off[1:] = np.cumsum(segs)
    seg = torch.from_numpy(off).cuda()
    s = torch.cuda.current_stream().cuda_stream
    h = torch.empty((rows, 2 * f), dtype=torch.bfloat16, device="cuda")
    act = torch.empty((rows, f), dtype=torch.bfloat16, device="cuda")
    y = torch.empty((rows, d), dtype=torch.bfloat16, device="cuda")
    assert lib.hm_grouped_ffn_fwd(x.data_ptr(), rows, seg.data_ptr(), E, w_ug.data_ptr(), w_d.data_ptr(), d, f,
                                  h.data_ptr(), act.data_ptr(), y.data_ptr(), 0, s) == 0
    dh = torch.empty_like(h)
    dx = torch.empty_like(x)
    dw_ug, dw_d = torch.empty_like(w_ug), torch.empty_like(w_d)
    nws = 2 * lib.hm_grouped_gemm_workspace_bytes(_native.GEMM_WGRAD, E)
    ws = torch.empty((nws + 128,), dtype=torch.uint8, device="cuda")
    wsp = ws.data_ptr() + (-ws.data_ptr()) % 128
    assert lib.hm_grouped_ffn_bwd(dy.data_ptr(), x.data_ptr(), h.data_ptr(), act.data_ptr(), rows, seg.data_ptr(),
                                  E, w_ug.data_ptr(), w_d.data_ptr(), d, f, dh.data_ptr(), dx.data_ptr(),
                                  dw_ug.data_ptr(), dw_d.data_ptr(), wsp, 0, s) == 0
    y2, h2, act2 = ops.grouped_ffn_fwd(x, seg, w_ug, w_d)
    dx2, dw_ug2, dw_d2 = ops.grouped_ffn_bwd(dy, x, h2, act2, seg, w_ug, w_d)
    torch.cuda.synchronize()
    for a, b in ((y, y2), (h, h2), (act, act2), (dx, dx2), (dw_ug, dw_ug2), (dw_d, dw_d2)):
        assert torch.equal(a, b)
    wg_, wu_ = ops.split_gate_up(w_ug.float().cpu())
    xr = x.float().cpu().requires_grad_()
    yr = orc.expert_ffn(xr, off, wg_, wu_, w_d.float().cpu())
    yr.backward(dy.float().cpu())
    assert orc.rel_err(y, yr) < TOL_ACT and orc.rel_err(dx, xr.grad) < TOL_ACT
