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
