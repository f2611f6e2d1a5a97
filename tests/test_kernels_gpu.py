"""GPU parity tests of the native kernels against the CPU oracle (run on a B200).

Bars: routing indices, counts, offsets, row maps and the permuted rows are
BIT-EXACT; gate weights within 1e-5 abs; expert outputs / combine / dX within relative
Frobenius error 1e-2 of the fp32 oracle fed the same bf16 inputs; weight grads within 2e-2.
"""

import numpy as np
import pytest
import torch

from oracle import moe_oracle as orc
from paper_2504_03871_b200 import ops
from paper_2504_03871_b200.configs import C1, C2, C3, LayerConfig, make_inputs, with_tokens

pytestmark = pytest.mark.gpu

TOL_ACT = 1e-2
TOL_W = 2e-2
TOL_GATE = 1e-5

ROUTER_CASES = [
    C1,
    with_tokens(C2, 1024),
    with_tokens(C3, 1536),
    LayerConfig("ragged", E=16, k=4, d=512, f=256, T=1000),
    LayerConfig("E256", E=256, k=8, d=256, f=128, T=777),
    LayerConfig("T1", E=8, k=2, d=256, f=128, T=1),
]


def _route_gpu(inp, cfg):
    return ops.router_topk(inp.x.cuda(), inp.wg.cuda(), cfg.k)


@pytest.mark.parametrize("cfg", ROUTER_CASES, ids=lambda c: c.name)
def test_router_bit_exact(cfg):
    inp = make_inputs(cfg, seed=1)
    ref = orc.route(inp.x.float().numpy(), inp.wg.float().numpy(), cfg.k)
    r = _route_gpu(inp, cfg)
    torch.cuda.synchronize()
    logits = r.logits.cpu().numpy()
    assert np.array_equal(logits.view(np.uint32), ref.logits.view(np.uint32)), "logits not bit-exact"
    assert np.array_equal(r.idx.cpu().numpy(), ref.idx)
    assert np.array_equal(r.counts.cpu().numpy(), ref.counts)
    assert np.array_equal(r.offsets.cpu().numpy(), ref.offsets)
    assert np.abs(r.w.cpu().numpy() - ref.w).max() <= TOL_GATE


@pytest.mark.parametrize("cfg", ROUTER_CASES[:3], ids=lambda c: c.name)
def test_router_with_bias_bit_exact(cfg):
    from paper_2504_03871_b200.configs import zipf_bias

    inp = make_inputs(cfg, seed=4)
    bias = np.asarray(zipf_bias(cfg.E, 1.0), dtype=np.float32)
    ref = orc.route(inp.x.float().numpy(), inp.wg.float().numpy(), cfg.k, bias=bias)
    r = ops.router_topk(inp.x.cuda(), inp.wg.cuda(), cfg.k, torch.from_numpy(bias).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(r.logits.cpu().numpy().view(np.uint32), ref.logits.view(np.uint32))
    assert np.array_equal(r.idx.cpu().numpy(), ref.idx)
    assert np.array_equal(r.counts.cpu().numpy(), ref.counts)


@pytest.mark.parametrize("cfg", [C2, C3], ids=lambda c: c.name)
def test_full_size_routing_and_permutation_bit_exact(cfg):
    """Full BASELINE sizes (T=16384): the C restatement of the router checks every index,
    count, offset and row map; the permuted rows are checked as a gather of x."""
    g = torch.Generator().manual_seed(21)
    x = (torch.randn((cfg.T, cfg.d), generator=g)).to(torch.bfloat16)
    wg = (torch.randn((cfg.d, cfg.E), generator=g) * cfg.d ** -0.5).to(torch.bfloat16)
    ref = orc.route_c(x, wg, cfg.k)
    xc = x.cuda()
    r = ops.router_topk(xc, wg.cuda(), cfg.k)
    x_perm, row_src, row_of = ops.dispatch_permute(xc, r)
    torch.cuda.synchronize()
    assert np.array_equal(r.logits.cpu().numpy().view(np.uint32), ref.logits.view(np.uint32))
    assert np.array_equal(r.idx.cpu().numpy(), ref.idx)
    assert np.array_equal(r.counts.cpu().numpy(), ref.counts)
    assert np.array_equal(r.offsets.cpu().numpy(), ref.offsets)
    assert np.array_equal(row_src.cpu().numpy(), ref.row_src)
    assert np.array_equal(row_of.cpu().numpy(), ref.row_of)
    assert torch.equal(x_perm, xc[row_src.long()])
    assert int(r.offsets[-1]) == cfg.T * cfg.k  # dropless: every copy placed


@pytest.mark.parametrize("cfg", ROUTER_CASES, ids=lambda c: c.name)
def test_permute_bit_exact(cfg):
    inp = make_inputs(cfg, seed=2)
    ref = orc.route(inp.x.float().numpy(), inp.wg.float().numpy(), cfg.k)
    x = inp.x.cuda()
    r = _route_gpu(inp, cfg)
    x_perm, row_src, row_of = ops.dispatch_permute(x, r)
    torch.cuda.synchronize()
    assert np.array_equal(row_src.cpu().numpy(), ref.row_src)
    assert np.array_equal(row_of.cpu().numpy(), ref.row_of)
    expect = inp.x[torch.from_numpy(ref.row_src.astype(np.int64))]
    assert torch.equal(x_perm.cpu(), expect)
    # unpermute-sum of the permuted copy is k * x exactly representable? compare in fp32
    dx = ops.unpermute_sum(x_perm, row_of).float().cpu()
    assert orc.rel_err(dx, cfg.k * inp.x.float()) < 1e-2


@pytest.mark.parametrize("cfg", ROUTER_CASES[:4], ids=lambda c: c.name)
def test_combine_and_bwd(cfg):
    inp = make_inputs(cfg, seed=3)
    r = _route_gpu(inp, cfg)
    x = inp.x.cuda()
    _, _, row_of = ops.dispatch_permute(x, r)
    g = torch.Generator().manual_seed(5)
    y_perm = torch.randn((cfg.T * cfg.k, cfg.d), generator=g).to(torch.bfloat16)
    dy = inp.dy
    y = ops.combine(y_perm.cuda(), row_of, r.w)
    dy_perm, dw = ops.combine_bwd(dy.cuda(), y_perm.cuda(), row_of, r.w)
    torch.cuda.synchronize()
    ro = row_of.long().cpu()
    w = r.w.cpu()
    yp = y_perm.float()
    y_ref = (yp[ro.reshape(-1)].reshape(cfg.T, cfg.k, -1) * w[:, :, None]).sum(1)
    assert orc.rel_err(y, y_ref) < TOL_ACT
    dyp_ref = torch.zeros_like(yp)
    dyp_ref[ro.reshape(-1)] = (w[:, :, None] * dy.float()[:, None, :]).reshape(-1, cfg.d)
    assert orc.rel_err(dy_perm, dyp_ref) < TOL_ACT
    dw_ref = (yp[ro.reshape(-1)].reshape(cfg.T, cfg.k, -1) * dy.float()[:, None, :]).sum(-1)
    assert orc.rel_err(dw, dw_ref) < 1e-4


def _ragged_offsets(counts):
    off = np.zeros(len(counts) + 1, dtype=np.int32)
    off[1:] = np.cumsum(counts)
    return off


GEMM_SEGS = [
    [128, 256],
    [1, 0, 130, 127, 300, 0, 64, 2],
    [0, 0, 0, 700],
    [513],
]


@pytest.mark.parametrize("segs", GEMM_SEGS, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("df", [(256, 384), (512, 128)], ids=lambda p: f"d{p[0]}f{p[1]}")
def test_grouped_ffn_vs_fp32(segs, df):
    d, f = df
    E = len(segs)
    rows = int(sum(segs))
    g = torch.Generator().manual_seed(11)
    bf = lambda *s, std=1.0: (torch.randn(s, generator=g) * std).to(torch.bfloat16)
    x_perm = bf(rows, d)
    w_gate, w_up = bf(E, f, d, std=d ** -0.5), bf(E, f, d, std=d ** -0.5)
    w_down = bf(E, d, f, std=f ** -0.5)
    dy = bf(rows, d)
    off = _ragged_offsets(segs)
    w_ug = ops.interleave_gate_up(w_gate, w_up)
    seg = torch.from_numpy(off).cuda()
    y, h, act = ops.grouped_ffn_fwd(x_perm.cuda(), seg, w_ug.cuda(), w_down.cuda())
    dx, dw_ug, dw_d = ops.grouped_ffn_bwd(dy.cuda(), x_perm.cuda(), h, act, seg, w_ug.cuda(),
                                          w_down.cuda())
    torch.cuda.synchronize()
    # fp32 reference with autograd
    xr = x_perm.float().requires_grad_()
    wgr = w_gate.float().requires_grad_()
    wur = w_up.float().requires_grad_()
    wdr = w_down.float().requires_grad_()
    yr = orc.expert_ffn(xr, off, wgr, wur, wdr)
    yr.backward(dy.float())
    assert orc.rel_err(y, yr) < TOL_ACT
    assert orc.rel_err(dx, xr.grad) < TOL_ACT
    dg, du = ops.split_gate_up(dw_ug.cpu())
    for e in range(E):
        if segs[e] == 0:
            assert torch.count_nonzero(dg[e]) == 0 and torch.count_nonzero(dw_d[e]) == 0
    assert orc.rel_err(dg, wgr.grad) < TOL_W
    assert orc.rel_err(du, wur.grad) < TOL_W
    assert orc.rel_err(dw_d, wdr.grad) < TOL_W
    # fp32 accumulation variant: two accumulations of the same micro-batch = 2x the gradient
    gw_ug = torch.zeros(w_ug.shape, dtype=torch.float32, device="cuda")
    gw_d = torch.zeros(w_down.shape, dtype=torch.float32, device="cuda")
    for _ in range(2):
        dx2 = ops.grouped_ffn_bwd_acc(dy.cuda(), x_perm.cuda(), h, act, seg, w_ug.cuda(),
                                      w_down.cuda(), gw_ug, gw_d)
    torch.cuda.synchronize()
    assert torch.equal(dx2.cpu(), dx.cpu())
    ag, au = ops.split_gate_up(gw_ug.cpu())
    assert orc.rel_err(ag, 2 * wgr.grad) < TOL_W
    assert orc.rel_err(au, 2 * wur.grad) < TOL_W
    assert orc.rel_err(gw_d, 2 * wdr.grad) < TOL_W


def test_grouped_wgrad_multi_segment_matches_sum():
    """One K-concatenated weight-gradient GEMM over R micro-batches == the fp32 sum of the
    per-micro-batch gradients (ragged and empty segments included)."""
    d, f = 256, 384
    seg_sets = [[100, 0, 257], [0, 0, 64], [31, 500, 1], [0, 0, 0]]
    E = 3
    g = torch.Generator().manual_seed(8)
    bf = lambda *s, std=1.0: (torch.randn(s, generator=g) * std).to(torch.bfloat16).cuda()  # noqa: E731
    dhs, xs, segs = [], [], []
    for segs_j in seg_sets:
        rows = max(sum(segs_j), 1)
        dhs.append(bf(rows, 2 * f))
        xs.append(bf(rows, d))
        segs.append(_ragged_offsets(segs_j).tolist())
    seg_multi = torch.tensor(segs, dtype=torch.int32, device="cuda")
    out = torch.zeros((E, 2 * f, d), dtype=torch.float32, device="cuda")
    ops.grouped_wgrad_multi(dhs, xs, seg_multi, out, accumulate=True)
    ref = torch.zeros((E, 2 * f, d), dtype=torch.float32)
    for dh, x, so in zip(dhs, xs, segs):
        for e in range(E):
            a, b = so[e], so[e + 1]
            ref[e] += dh[a:b].float().cpu().t() @ x[a:b].float().cpu()
    torch.cuda.synchronize()
    assert orc.rel_err(out, ref) < 1e-3


def test_grouped_ffn_capacity_cap_matches_dynamic_schedule():
    """max_ctas (persistent, static tile striding: the capacity-weight emulation) and the
    default dynamic cluster-launch-control schedule compute identical results."""
    segs = [300, 0, 1000, 257, 31, 700]
    d, f = 512, 384
    E = len(segs)
    g = torch.Generator().manual_seed(5)
    bf = lambda *s, std=1.0: (torch.randn(s, generator=g) * std).to(torch.bfloat16).cuda()  # noqa: E731
    x = bf(sum(segs), d)
    w_ug = bf(E, 2 * f, d, std=d ** -0.5)
    w_d = bf(E, d, f, std=f ** -0.5)
    dy = bf(sum(segs), d)
    seg = torch.from_numpy(_ragged_offsets(segs)).cuda()
    outs = []
    for cap in (0, 20, 7):
        y, h, act = ops.grouped_ffn_fwd(x, seg, w_ug, w_d, max_ctas=cap)
        dx, dwu, dwd = ops.grouped_ffn_bwd(dy, x, h, act, seg, w_ug, w_d, max_ctas=cap)
        outs.append((y, h, act, dx, dwu, dwd))
    torch.cuda.synchronize()
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert torch.equal(a, b)


@pytest.mark.parametrize("cfg", [with_tokens(C1, 1024), LayerConfig("c3ish", 16, 4, 512, 384, 700)],
                         ids=lambda c: c.name)
def test_moe_layer_fwd_bwd(cfg):
    from paper_2504_03871_b200.layer import moe_forward

    inp = make_inputs(cfg, seed=7)
    w_ug = ops.interleave_gate_up(inp.w_gate, inp.w_up)
    x = inp.x.cuda().requires_grad_()
    wg = inp.wg.cuda().requires_grad_()
    wug = w_ug.cuda().requires_grad_()
    wd = inp.w_down.cuda().requires_grad_()
    y, idx = moe_forward(x, wg, wug, wd, cfg.k)
    y.backward(inp.dy.cuda())
    torch.cuda.synchronize()
    ref = orc.moe_layer(inp.x, inp.wg, w_ug, inp.w_down, cfg.k, dy=inp.dy)
    assert np.array_equal(idx.cpu().numpy(), ref["routing"].idx)
    assert orc.rel_err(y, ref["y"]) < TOL_ACT
    assert orc.rel_err(x.grad, ref["dx"]) < TOL_ACT
    assert orc.rel_err(wg.grad, ref["dwg"]) < TOL_W
    dg, du = ops.split_gate_up(wug.grad.cpu())
    assert orc.rel_err(dg, ref["dw_gate"]) < TOL_W
    assert orc.rel_err(du, ref["dw_up"]) < TOL_W
    assert orc.rel_err(wd.grad, ref["dw_down"]) < TOL_W


@pytest.mark.parametrize("segs,M,N", [
    ([1, 0, 130, 127, 300, 0, 64, 2], 256, 512),
    ([100] * 7 + [24], 512, 128),
    ([4096, 4000, 4200, 3900], 8192, 4096),
    ([0, 0, 1, 700], 768, 256),
])
def test_device_expert_maps_match_host(segs, M, N):
    """The per-expert TMA views that the wgrad GEMM builds on the device (tensormap.replace of
    the whole-buffer maps) are byte-identical to the driver's own encoding of the same views."""
    import ctypes

    from paper_2504_03871_b200 import _native

    lib = _native.load()
    fn = lib.hm_debug_expert_maps
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4 + [ctypes.c_void_p]
    E = len(segs)
    rows = max(sum(segs), 1)
    off = _ragged_offsets(segs)
    seg = torch.from_numpy(off).cuda()
    a = torch.empty((rows, M), dtype=torch.bfloat16, device="cuda")
    b = torch.empty((rows, N), dtype=torch.bfloat16, device="cuda")
    buf = (ctypes.c_ubyte * (4 * E * 128))()
    assert fn(a.data_ptr(), b.data_ptr(), seg.data_ptr(), E, rows, M, N, buf) == 0
    arr = np.frombuffer(bytes(buf), dtype=np.uint8).reshape(2, E, 2, 128)
    for e in range(E):
        for o in range(2):
            assert np.array_equal(arr[0, e, o], arr[1, e, o]), (e, o, np.nonzero(arr[0, e, o] != arr[1, e, o]))


def test_grouped_ffn_full_c2_sampled_rows():
    """All six K3 GEMMs at the full C2 shape (E=8, d=4096, f=14336, 32768 routed rows in ragged
    experts) — the wide tiles with early accumulator release, the narrow SwiGLU backward — checked
    on sampled rows / weight rows against a plain PyTorch fp32 reference computed on the GPU from
    the same bf16 operands."""
    E, d, f = 8, 4096, 14336
    segs = [4096 + 517, 4096 - 517, 3000, 5192, 4096, 4096 + 255, 4096 - 255, 4096]
    rows = sum(segs)
    g = torch.Generator(device="cuda").manual_seed(3)
    bf = lambda *s, std=1.0: (torch.randn(s, generator=g, device="cuda") * std).to(torch.bfloat16)  # noqa: E731
    x = bf(rows, d)
    w_ug = bf(E, 2 * f, d, std=d ** -0.5)
    w_d = bf(E, d, f, std=f ** -0.5)
    dy = bf(rows, d)
    off = _ragged_offsets(segs)
    seg = torch.from_numpy(off).cuda()
    y, h, act = ops.grouped_ffn_fwd(x, seg, w_ug, w_d)
    dx, dw_ug, dw_d = ops.grouped_ffn_bwd(dy, x, h, act, seg, w_ug, w_d)
    torch.cuda.synchronize()
    wg_, wu_ = ops.split_gate_up(w_ug)
    sel = torch.randint(0, rows, (96,), generator=torch.Generator().manual_seed(0)).tolist()
    sel += [off[e] for e in range(E)] + [off[e + 1] - 1 for e in range(E)]  # expert boundaries
    for r in sel:
        e = int(np.searchsorted(off, r, side="right") - 1)
        xr = x[r].float()
        gate = wg_[e].float() @ xr
        up = wu_[e].float() @ xr
        hq_g, hq_u = ops.split_gate_up(h[r].float().view(1, 2 * f, 1))  # saved gate / up (bf16)
        assert orc.rel_err(hq_g.reshape(-1), gate) < TOL_ACT
        assert orc.rel_err(hq_u.reshape(-1), up) < TOL_ACT
        a_ref = torch.nn.functional.silu(gate) * up
        assert orc.rel_err(act[r].float(), a_ref) < TOL_ACT
        assert orc.rel_err(y[r].float(), w_d[e].float() @ act[r].float()) < TOL_ACT
        # backward from the kernel's own saved h (bf16) and the row's dY
        da = w_d[e].float().t() @ dy[r].float()
        gq, uq = hq_g.reshape(-1), hq_u.reshape(-1)
        sg = torch.sigmoid(gq)
        dgate = da * uq * sg * (1 + gq * (1 - sg))
        dup = da * gq * sg
        dx_ref = wg_[e].float().t() @ dgate + wu_[e].float().t() @ dup
        assert orc.rel_err(dx[r].float(), dx_ref) < TOL_ACT
    # weight gradients: sampled output rows of dW_d[e] and dW_ug[e] over the expert's rows
    for e in (0, 3, 7):
        a, b = int(off[e]), int(off[e + 1])
        for i in (0, 1234, d - 1):
            ref = dy[a:b, i].float() @ act[a:b].float()
            assert orc.rel_err(dw_d[e, i].float(), ref) < TOL_W
        for j in (0, 777, 2 * f - 1):
            # dW_ug[e][j] = sum over the expert's rows of dH[:, j] * x (interleaved gate|up
            # layout: 256-row blocks = 128 gate rows then 128 up rows), dH from the saved h
            blk, within = j // 256, j % 256
            is_up = within >= 128
            fcol = blk * 128 + (within - 128 if is_up else within)
            gq = h[a:b, blk * 256 + (within - 128 if is_up else within)].float()
            uq = h[a:b, blk * 256 + 128 + (within - 128 if is_up else within)].float()
            da = dy[a:b].float() @ w_d[e, :, fcol].float()
            sg = torch.sigmoid(gq)
            dcol = da * gq * sg if is_up else da * uq * sg * (1 + gq * (1 - sg))
            ref = dcol @ x[a:b].float()
            assert orc.rel_err(dw_ug[e, j].float(), ref) < TOL_W


def _with_env(name, fn):
    import os

    os.environ[name] = "1"
    try:
        return fn()
    finally:
        os.environ.pop(name, None)


def _bits(t):
    return t.view(torch.int32) if t.dtype == torch.float32 else t


@pytest.mark.parametrize("cfg", [with_tokens(C3, 1000), LayerConfig("E32", E=32, k=4, d=256, f=128, T=333),
                                 with_tokens(C1, 999)], ids=lambda c: c.name)
def test_topk_thread_per_token_matches_warp_kernel(cfg):
    """router_topk_lane_kernel (E <= 64) vs router_topk_kernel (HM_TOPK_WARP): every routing
    output bitwise equal, including an all-tie row (zero input) and an all-NaN row."""
    import os

    inp = make_inputs(cfg, seed=7)
    x = inp.x.cuda().clone()
    x[1] = 0
    x[2] = float("nan")
    wg = inp.wg.cuda()
    os.environ["HM_ROUTER_UNFUSED"] = "1"
    try:
        a = ops.router_topk(x, wg, cfg.k)
        b = _with_env("HM_TOPK_WARP", lambda: ops.router_topk(x, wg, cfg.k))
    finally:
        os.environ.pop("HM_ROUTER_UNFUSED", None)
    for name in ("idx", "w", "counts", "offsets"):
        assert torch.equal(_bits(getattr(a, name)), _bits(getattr(b, name))), name
    n = ((cfg.T + 63) // 64) * cfg.E  # the table's last element is the fused kernel's counter
    assert torch.equal(a.chunk_base[:n], b.chunk_base[:n])


@pytest.mark.parametrize("cfg", [with_tokens(C3, 777), with_tokens(C1, 500)], ids=lambda c: c.name)
def test_unpermute_router_bwd_variants_bitwise_equal(cfg):
    """unpermute_router_bwd_kernel (v1) and unpermute_router_bwd2_kernel (v2 prefetch / v3):
    dx, dlogit and dWg bitwise equal."""
    inp = make_inputs(cfg, seed=8)
    x, wg = inp.x.cuda(), inp.wg.cuda()
    r = ops.router_topk(x, wg, cfg.k)
    xp, _, row_of = ops.dispatch_permute(x, r)
    g = torch.Generator(device="cuda").manual_seed(3)
    dxp = torch.randn(xp.shape, generator=g, device="cuda").to(xp.dtype)
    dw = torch.randn(r.w.shape, generator=g, device="cuda")
    wg_t = ops.transpose_bf16(wg)
    outs = {v: _with_env("HM_UNPERMUTE_" + v, lambda: ops.router_bwd(dxp, row_of, r, dw, xp, wg_t))
            for v in ("V1", "V2", "V3")}
    for v in ("V2", "V3"):
        for a, b in zip(outs["V1"], outs[v]):
            assert torch.equal(_bits(a), _bits(b)), v


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs in one process")
def test_one_process_two_devices():
    """The library keeps no per-device state that only the first device gets: the dynamic shared
    memory opt-ins of the router, the grouped GEMM and the router weight gradient are made on each
    device's context, so one process can run the layer on cuda:0, then cuda:1, then cuda:0."""
    from paper_2504_03871_b200.layer import moe_forward

    cfg = LayerConfig("two_dev", E=8, k=2, d=512, f=384, T=700)
    inp = make_inputs(cfg, seed=11)
    w_ug = ops.interleave_gate_up(inp.w_gate, inp.w_up)
    ref = orc.moe_layer(inp.x, inp.wg, w_ug, inp.w_down, cfg.k, dy=inp.dy)
    for dev in ("cuda:0", "cuda:1", "cuda:0"):
        with torch.cuda.device(dev):
            x = inp.x.to(dev).requires_grad_()
            wg = inp.wg.to(dev).requires_grad_()
            wug = w_ug.to(dev).requires_grad_()
            wd = inp.w_down.to(dev).requires_grad_()
            y, idx = moe_forward(x, wg, wug, wd, cfg.k)
            y.backward(inp.dy.to(dev))
            torch.cuda.synchronize()
        assert np.array_equal(idx.cpu().numpy(), ref["routing"].idx), dev
        assert orc.rel_err(y, ref["y"]) < TOL_ACT, dev
        assert orc.rel_err(x.grad, ref["dx"]) < TOL_ACT, dev
        assert orc.rel_err(wd.grad, ref["dw_down"]) < TOL_W, dev


def test_ops_reject_wrong_dtype_and_layout():
    """The C ABI reads raw bytes: a wrong dtype, a CPU or a non-contiguous tensor is an error at
    the operator boundary, never a silent reinterpretation (the reference raises ValueError /
    TypeError for bad inputs the same way)."""
    cfg = LayerConfig("dtype", E=8, k=2, d=256, f=128, T=64)
    inp = make_inputs(cfg, seed=3)
    x, wg = inp.x.cuda(), inp.wg.cuda()
    with pytest.raises(TypeError):
        ops.router_topk(x.float(), wg, cfg.k)
    with pytest.raises(TypeError):
        ops.router_topk(x, wg.float(), cfg.k)
    with pytest.raises(ValueError):
        ops.router_topk(inp.x, wg, cfg.k)
    with pytest.raises(ValueError):
        ops.router_topk(x.t().contiguous().t(), wg, cfg.k)
    r = ops.router_topk(x, wg, cfg.k)
    xp, _, row_of = ops.dispatch_permute(x, r)
    with pytest.raises(TypeError):
        ops.combine(xp, row_of.long(), r.w)
    with pytest.raises(TypeError):
        ops.combine(xp, row_of, r.w.bfloat16())
    with pytest.raises(TypeError):
        ops.dispatch_permute(x.half(), r)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs in one process")
def test_ops_reject_tensor_on_other_device():
    cfg = LayerConfig("dev", E=8, k=2, d=256, f=128, T=64)
    inp = make_inputs(cfg, seed=3)
    with torch.cuda.device(0):
        with pytest.raises(ValueError, match="current CUDA device"):
            ops.router_topk(inp.x.to("cuda:1"), inp.wg.to("cuda:1"), cfg.k)


def test_moe_layer_module_batched_input_matches_oracle():
    """MoELayer (the nn.Module face of the layer) over a [batch, seq, d] input, and moe_forward
    over a strided view of the token rows, against the oracle."""
    from paper_2504_03871_b200.layer import MoELayer, moe_forward

    cfg = LayerConfig("module", E=8, k=2, d=512, f=384, T=600)
    inp = make_inputs(cfg, seed=5)
    w_ug = ops.interleave_gate_up(inp.w_gate, inp.w_up)
    ref = orc.moe_layer(inp.x, inp.wg, w_ug, inp.w_down, cfg.k, dy=inp.dy)
    layer = MoELayer(cfg.d, cfg.f, cfg.E, cfg.k).load(inp.wg.cuda(), inp.w_gate.cuda(), inp.w_up.cuda(),
                                                      inp.w_down.cuda())
    x = inp.x.cuda().view(3, 200, cfg.d).requires_grad_()
    y = layer(x)
    assert y.shape == x.shape
    y.backward(inp.dy.cuda().view(3, 200, cfg.d))
    torch.cuda.synchronize()
    assert orc.rel_err(y.reshape(cfg.T, cfg.d), ref["y"]) < TOL_ACT
    assert orc.rel_err(x.grad.reshape(cfg.T, cfg.d), ref["dx"]) < TOL_ACT
    assert orc.rel_err(layer.wg.grad, ref["dwg"]) < TOL_W
    assert orc.rel_err(layer.w_down.grad, ref["dw_down"]) < TOL_W
    # a column-strided view of the token rows is made contiguous at the boundary
    wide = torch.zeros((cfg.T, 2 * cfg.d), dtype=torch.bfloat16, device="cuda")
    wide[:, : cfg.d] = inp.x.cuda()
    y2, idx2 = moe_forward(wide[:, : cfg.d], layer.wg.detach(), layer.w_ug.detach(), layer.w_down.detach(), cfg.k)
    assert np.array_equal(idx2.cpu().numpy(), ref["routing"].idx)
    assert torch.equal(y2, y.detach().reshape(cfg.T, cfg.d))


@pytest.mark.parametrize("groupm", [1, 3, -1, -3, -8], ids=lambda g: f"groupm{g}")
def test_grouped_ffn_any_raster_is_bitwise_equal(groupm):
    """The raster (tile order) only changes which CTA computes a tile, never its arithmetic: every
    row-grouped (g > 0) and transposed (g < 0) raster gives the default's bits, on ragged experts
    with several m- and n-tiles per expert."""
    from paper_2504_03871_b200 import _native

    lib = _native.load()
    segs = [700, 0, 513, 1, 256, 300]
    d, f = 1024, 640  # 2 wide n-tiles for the d-wide GEMMs, 3 for the 2f-wide up+gate
    E, rows = len(segs), sum(segs)
    g = torch.Generator().manual_seed(5)
    bf = lambda *s, std=1.0: (torch.randn(s, generator=g) * std).to(torch.bfloat16).cuda()  # noqa: E731
    x_perm, dy = bf(rows, d), bf(rows, d)
    w_ug, w_d = bf(E, 2 * f, d, std=d ** -0.5), bf(E, d, f, std=f ** -0.5)
    seg = torch.from_numpy(_ragged_offsets(segs)).cuda()

    def run():
        y, h, act = ops.grouped_ffn_fwd(x_perm, seg, w_ug, w_d)
        dx, dw_ug, dw_d = ops.grouped_ffn_bwd(dy, x_perm, h, act, seg, w_ug, w_d)
        torch.cuda.synchronize()
        return [t.clone() for t in (y, h, act, dx, dw_ug, dw_d)]

    ref = run()
    lib.hm_debug_set_gemm_groupm(-1, groupm)
    try:
        got = run()
    finally:
        lib.hm_debug_set_gemm_groupm(-1, 0)
    for a, b in zip(ref, got):
        assert torch.equal(a, b)


@pytest.mark.parametrize("k", [1, 2, 3, 6])
@pytest.mark.parametrize("d", [296, 1032])
def test_combine_any_width_vs_fp32(k, d):
    """K4 on widths that are not a multiple of 256 (nv = d / 8 column segments not a multiple of
    32 lanes, so the last group of in-flight segments is partial) against an fp32 reference."""
    T = 333
    g = torch.Generator().manual_seed(9)
    row_of = torch.randperm(T * k, generator=g).to(torch.int32).reshape(T, k)
    w = torch.softmax(torch.randn((T, k), generator=g), 1)
    y_perm = torch.randn((T * k, d), generator=g).to(torch.bfloat16)
    dy = torch.randn((T, d), generator=g).to(torch.bfloat16)
    y = ops.combine(y_perm.cuda(), row_of.cuda(), w.cuda())
    dy_perm, dw = ops.combine_bwd(dy.cuda(), y_perm.cuda(), row_of.cuda(), w.cuda())
    torch.cuda.synchronize()
    ro = row_of.long()
    yp = y_perm.float()
    y_ref = (yp[ro.reshape(-1)].reshape(T, k, -1) * w[:, :, None]).sum(1)
    assert orc.rel_err(y, y_ref) < TOL_ACT
    dyp_ref = torch.zeros_like(yp)
    dyp_ref[ro.reshape(-1)] = (w[:, :, None] * dy.float()[:, None, :]).reshape(-1, d)
    assert orc.rel_err(dy_perm, dyp_ref) < TOL_ACT
    dw_ref = (yp[ro.reshape(-1)].reshape(T, k, -1) * dy.float()[:, None, :]).sum(-1)
    assert orc.rel_err(dw, dw_ref) < 1e-4
