"""Single-GPU checks of the peer-memory transport kernels (the executor's ``transport="p2p"``):
each is run with its destinations on the local device, where the result must equal the
unfused kernel's output rearranged into the owners' receive layout (bit-exact for the row
moves; the GEMM row scatter bit-exact against the contiguous store of the same GEMM)."""

import numpy as np
import pytest
import torch

from paper_2504_03871_b200 import _native, ops
from paper_2504_03871_b200.configs import C1, LayerConfig, make_inputs

pytestmark = pytest.mark.gpu

CASES = [C1, LayerConfig("ragged", E=16, k=4, d=512, f=256, T=1000),
         LayerConfig("d6144", E=8, k=2, d=6144, f=256, T=300)]  # generic-width row copy


def _owner_layout(offsets, E, n_owner, pad=3):
    """Experts dealt round-robin to n_owner receive buffers; each buffer holds its experts'
    rows back to back after `pad` spare rows. Returns (dest_base index per expert, dest_start,
    rows per owner)."""
    owner = [e % n_owner for e in range(E)]
    start, fill = [0] * E, [pad] * n_owner
    for e in range(E):
        start[e] = fill[owner[e]]
        fill[owner[e]] += int(offsets[e + 1] - offsets[e])
    return owner, start, fill


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: c.name)
def test_dispatch_permute_p2p_matches_permute(cfg):
    inp = make_inputs(cfg, seed=11)
    x = inp.x.cuda()
    r = ops.router_topk(x, inp.wg.cuda(), cfg.k)
    x_perm, _, row_of = ops.dispatch_permute(x, r)
    off = r.offsets.cpu().numpy()
    owner, start, fill = _owner_layout(off, cfg.E, 3)
    bufs = [torch.full((n, cfg.d), 7.0, dtype=torch.bfloat16, device="cuda") for n in fill]
    base = torch.tensor([bufs[o].data_ptr() for o in owner], dtype=torch.uint64, device="cuda")
    st = torch.tensor(start, dtype=torch.int32, device="cuda")
    xp2, row_of2 = ops.dispatch_permute_p2p(x, r, base, st, keep_local=True)
    _, row_of3 = ops.dispatch_permute_p2p(x, r, base, st, keep_local=False)
    torch.cuda.synchronize()
    assert torch.equal(row_of2, row_of) and torch.equal(row_of3, row_of)
    assert torch.equal(xp2, x_perm)
    for e in range(cfg.E):
        n = int(off[e + 1] - off[e])
        got = bufs[owner[e]][start[e]:start[e] + n]
        assert torch.equal(got, x_perm[off[e]:off[e + 1]]), f"expert {e}"
    for b in bufs:  # the pad rows are untouched
        assert bool((b[:3] == 7.0).all())


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: c.name)
def test_combine_bwd_p2p_matches_combine_bwd(cfg):
    inp = make_inputs(cfg, seed=12)
    x = inp.x.cuda()
    r = ops.router_topk(x, inp.wg.cuda(), cfg.k)
    _, _, row_of = ops.dispatch_permute(x, r)
    y_perm = torch.randn((cfg.T * cfg.k, cfg.d), device="cuda").to(torch.bfloat16)
    dy = inp.dy.cuda()
    dy_perm, dw = ops.combine_bwd(dy, y_perm, row_of, r.w)
    off = r.offsets.cpu().numpy()
    owner, start, fill = _owner_layout(off, cfg.E, 2)
    bufs = [torch.zeros((n, cfg.d), dtype=torch.bfloat16, device="cuda") for n in fill]
    base = torch.tensor([bufs[o].data_ptr() for o in owner], dtype=torch.uint64, device="cuda")
    st = torch.tensor(start, dtype=torch.int32, device="cuda")
    dw2 = ops.combine_bwd_p2p(dy, y_perm, row_of, r, base, st)
    torch.cuda.synchronize()
    assert torch.allclose(dw2, dw, rtol=1e-5, atol=1e-5)
    for e in range(cfg.E):
        n = int(off[e + 1] - off[e])
        assert torch.equal(bufs[owner[e]][start[e]:start[e] + n], dy_perm[off[e]:off[e + 1]]), f"expert {e}"


@pytest.mark.parametrize("segs", [[128, 256], [1, 0, 130, 127, 300, 0, 64, 2]], ids=lambda s: "x".join(map(str, s)))
def test_gemm_row_scatter_matches_contiguous(segs):
    d, f = 256, 384
    E = len(segs)
    rows = sum(segs)
    off = np.zeros(E + 1, dtype=np.int32)
    off[1:] = np.cumsum(segs)
    seg = torch.from_numpy(off).cuda()
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((rows, d), generator=g, device="cuda").to(torch.bfloat16)
    w_ug = (torch.randn((E, 2 * f, d), generator=g, device="cuda") * d ** -0.5).to(torch.bfloat16)
    w_d = (torch.randn((E, d, f), generator=g, device="cuda") * f ** -0.5).to(torch.bfloat16)
    y, h, act = ops.grouped_ffn_fwd(x, seg, w_ug, w_d)
    # forward: row r of the down projection goes to dest row perm[r] of another buffer
    perm = torch.randperm(rows, generator=torch.Generator().manual_seed(0))
    dest = torch.zeros((rows + 5, d), dtype=torch.bfloat16, device="cuda")
    out_rows = (dest.data_ptr() + (perm + 5) * d * 2).to(torch.uint64).cuda()
    h2, act2 = ops.grouped_ffn_fwd_rows(x, seg, w_ug, w_d, out_rows)
    torch.cuda.synchronize()
    assert torch.equal(h2, h) and torch.equal(act2, act)
    assert torch.equal(dest[5:][perm.cuda()], y)
    assert bool((dest[:5] == 0).all())
    # backward data path: dX rows scattered the same way
    dy = torch.randn((rows, d), generator=g, device="cuda").to(torch.bfloat16)
    dx, dh = ops.grouped_ffn_bwd_data(dy, x, h, act, seg, w_ug, w_d)
    dest.zero_()
    dh2 = ops.grouped_ffn_bwd_data_rows(dy, x, h, act, seg, w_ug, w_d, out_rows)
    torch.cuda.synchronize()
    assert torch.equal(dh2, dh)
    assert torch.equal(dest[5:][perm.cuda()], dx)


def test_signal_then_wait_local_counters():
    flags = torch.zeros(8, dtype=torch.int32, device="cuda")
    base = flags.data_ptr()
    ops.signal_peers([base + 4 * i for i in range(0, 8, 2)])
    ops.signal_peers([base + 4 * i for i in range(0, 8, 2)])
    ops.wait_flags(base, 2, [2, 2, 2, 2])
    torch.cuda.synchronize()
    assert flags.tolist() == [2, 0, 2, 0, 2, 0, 2, 0]
    with pytest.raises(_native.NativeLibraryError):
        ops.signal_peers([base] * 9)  # more than kMaxPeers


@pytest.mark.parametrize("M,N,offload,E", [(1, 1, 0, 8), (2, 2, 1, 8), (4, 4, 1, 8), (2, 2, 0, 64), (3, 1, 0, 6)])
def test_device_layout_matches_host_layout(M, N, offload, E):
    """hm_zp_layout (device receive layout, no host read of the counts) against the executor's
    host layout (``_recv_layout`` / ``p2p_dispatch_dest`` / ``p2p_return_rows``) on random counts
    with empty segments, for every rank of the exchange; plus the pool bump allocation, the GEMM
    row shifts and the overflow flag."""
    from paper_2504_03871_b200.executor import ZpExecutor, expert_owners, p2p_dispatch_dest, p2p_return_rows

    W = M + N
    owners = expert_owners(E, M, N, offload)
    rng = np.random.default_rng(M * 100 + N * 10 + E)
    counts_all = [[int(c) for c in rng.integers(0, 300, size=E)] for _ in range(M)]
    counts_all[0][0] = 0
    counts_all[-1][E - 1] = 0

    class _Ex:
        s = type("S", (), {"E": E})()
        st = type("St", (), {"owners": [owners]})()

    ex = _Ex()
    ex.M = M
    lay = {o: ZpExecutor._recv_layout(ex, 1, counts_all, o) for o in range(W)}
    send_off = {a: ZpExecutor._send_offsets(ex, counts_all[a]) for a in range(M)}
    cnt = torch.zeros((W, E), dtype=torch.int32)
    cnt[:M] = torch.tensor(counts_all, dtype=torch.int32)
    cnt = cnt.cuda()
    own_t = torch.tensor(owners, dtype=torch.int32, device="cuda")
    rb, dx_delta = 4096 * 2, 123456 * 16
    y_base = torch.tensor([(a + 1) << 32 for a in range(M)], dtype=torch.int64, device="cuda")
    cap = max(lay[o][0][-1] for o in range(W)) + 7
    for me in range(W):
        n_own = sum(1 for o in owners if o == me)
        dest_start = torch.full((E,), -1, dtype=torch.int32, device="cuda")
        seg = torch.full((max(n_own, 1) + 1,), -1, dtype=torch.int32, device="cuda")
        ory = torch.zeros((cap,), dtype=torch.int64, device="cuda")
        orx = torch.zeros((cap,), dtype=torch.int64, device="cuda")
        shifts = torch.zeros((2, 8), dtype=torch.int32, device="cuda")
        top = torch.zeros((1,), dtype=torch.int32, device="cuda")
        err = torch.zeros((1,), dtype=torch.int32, device="cuda")
        seg_h, pos = lay[me]
        total = seg_h[-1]
        for call in range(2):  # two micro-batches of the same counts: bump allocation
            ops.zp_layout(cnt, M, own_t, me, n_own, cap, y_base, dx_delta, rb, dest_start, seg, ory, orx,
                          shifts[call], top, 1000, 2 * total + 5, err)
        torch.cuda.synchronize()
        assert int(err.item()) == 0
        if me < M:
            _, ds = p2p_dispatch_dest(owners, {o: lay[o][1] for o in range(W)}, me, E)
            assert dest_start.tolist() == ds
        if n_own:
            assert seg[:n_own + 1].tolist() == seg_h
            ranks, rows = p2p_return_rows(pos, send_off)
            want = y_base.cpu().numpy()[ranks] + rows * rb
            assert np.array_equal(ory[:total].cpu().numpy(), want)
            assert np.array_equal(orx[:total].cpu().numpy(), want + dx_delta)
            for call, f in ((0, 1000), (1, 1000 + total)):
                assert shifts[call].tolist() == [0, f, f, 0, 0, f, f, 0]
            assert int(top.item()) == 2 * total
            # a third micro-batch overflows the pool region: flagged, segments emptied
            if total > 5:
                ops.zp_layout(cnt, M, own_t, me, n_own, cap, y_base, dx_delta, rb, dest_start, seg, ory, orx,
                              shifts[0], top, 1000, 2 * total + 5, err)
                torch.cuda.synchronize()
                assert int(err.item()) == 1 and int(top.item()) == 2 * total
                assert seg[:n_own + 1].tolist() == [0] * (n_own + 1)


@pytest.mark.parametrize("segs", [[128, 256], [1, 0, 130, 127, 300, 0, 64, 2]], ids=lambda s: "x".join(map(str, s)))
def test_pool_placed_ffn_matches_contiguous(segs):
    """The device-layout expert FFN (h / act / dH at a device-given pool row, receive slot padded
    to its capacity, outputs scattered by out_rows, weight gradients with per-segment pool shifts)
    against the contiguous per-micro-batch path: bitwise equal."""
    d, f = 256, 384
    E = len(segs)
    rows = sum(segs)
    cap = rows + 37
    off = np.zeros(E + 1, dtype=np.int32)
    off[1:] = np.cumsum(segs)
    seg = torch.from_numpy(off).cuda()
    g = torch.Generator(device="cuda").manual_seed(5)
    x_slot = torch.randn((cap, d), generator=g, device="cuda").to(torch.bfloat16)
    dy_slot = torch.randn((cap, d), generator=g, device="cuda").to(torch.bfloat16)
    x, dy = x_slot[:rows].contiguous(), dy_slot[:rows].contiguous()
    w_ug = (torch.randn((E, 2 * f, d), generator=g, device="cuda") * d ** -0.5).to(torch.bfloat16)
    w_d = (torch.randn((E, d, f), generator=g, device="cuda") * f ** -0.5).to(torch.bfloat16)
    y_ref, h_ref, act_ref = ops.grouped_ffn_fwd(x, seg, w_ug, w_d)
    dx_ref, dh_ref = ops.grouped_ffn_bwd_data(dy, x, h_ref, act_ref, seg, w_ug, w_d)
    gw_ug_ref = torch.zeros((E, 2 * f, d), dtype=torch.float32, device="cuda")
    gw_d_ref = torch.zeros((E, d, f), dtype=torch.float32, device="cuda")
    ops.grouped_wgrad_multi([dh_ref], [x], seg.view(1, -1), gw_ug_ref)
    ops.grouped_wgrad_multi([dy], [act_ref], seg.view(1, -1), gw_d_ref)
    # pool placement: this micro-batch at pool row 300 of a layer region starting at row 200
    base_l, f_row, pool = 200, 300, 300 + rows + 50
    h_pool = torch.zeros((pool, 2 * f), dtype=torch.bfloat16, device="cuda")
    act_pool = torch.zeros((pool, f), dtype=torch.bfloat16, device="cuda")
    dh_buf = torch.zeros((pool - base_l, 2 * f), dtype=torch.bfloat16, device="cuda")
    shifts = torch.tensor([0, f_row, f_row, 0, 0, f_row, f_row, 0], dtype=torch.int32, device="cuda")
    perm = torch.randperm(rows, generator=torch.Generator().manual_seed(1))
    y_dest = torch.zeros((rows + 3, d), dtype=torch.bfloat16, device="cuda")
    dx_dest = torch.zeros((rows + 3, d), dtype=torch.bfloat16, device="cuda")
    ory = torch.zeros((cap,), dtype=torch.int64, device="cuda")
    orx = torch.zeros((cap,), dtype=torch.int64, device="cuda")
    ory[:rows] = (y_dest.data_ptr() + (perm + 3) * d * 2).cuda()
    orx[:rows] = (dx_dest.data_ptr() + (perm + 3) * d * 2).cuda()
    ops.grouped_ffn_fwd_pool(x_slot, seg, w_ug, w_d, h_pool, act_pool, shifts, ory, cap)
    dh_ptr = dh_buf.data_ptr() - base_l * 2 * f * 2
    ops.grouped_ffn_bwd_data_pool(dy_slot, seg, w_ug, w_d, h_pool, dh_ptr, pool, shifts, orx, cap)
    gw_ug = torch.zeros_like(gw_ug_ref)
    gw_d = torch.zeros_like(gw_d_ref)
    seg2 = seg.view(1, -1).contiguous()
    ops.grouped_wgrad_multi_shifted([dh_ptr], [x_slot.data_ptr()], 2 * f, d, seg2, gw_ug, shift_a=shifts[1:2],
                                    shift_stride=8)
    ops.grouped_wgrad_multi_shifted([dy_slot.data_ptr()], [act_pool.data_ptr()], d, f, seg2, gw_d,
                                    shift_b=shifts[1:2], shift_stride=8)
    torch.cuda.synchronize()
    assert torch.equal(h_pool[f_row:f_row + rows], h_ref) and torch.equal(act_pool[f_row:f_row + rows], act_ref)
    assert bool((h_pool[:f_row] == 0).all()) and bool((h_pool[f_row + rows:] == 0).all())
    assert torch.equal(y_dest[3:][perm.cuda()], y_ref)
    assert torch.equal(dh_buf[f_row - base_l:f_row - base_l + rows], dh_ref)
    assert torch.equal(dx_dest[3:][perm.cuda()], dx_ref)
    assert torch.equal(gw_ug, gw_ug_ref) and torch.equal(gw_d, gw_d_ref)
