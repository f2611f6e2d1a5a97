"""Single-GPU MoE expert layer built from the native kernels (router -> permute -> grouped
SwiGLU FFN -> combine), forward and backward as one ``torch.autograd.Function``.

This is the computation the reference's ZP task chain ATTN_F -> DISP_F -> EXP_F -> COMB_F
(and the mirrored backward) stands for (``/root/reference/pkg/src/zpsim/taskgraph.py:453-502``)
when attention and experts share one device: no all-to-all, one expert group of E experts.
"""

from __future__ import annotations

import torch

from . import ops


def router_weight_t(wg: torch.Tensor) -> torch.Tensor:
    """Wg^T ([E, d], the router backward's layout), kept on the weight tensor itself and rebuilt
    only when the weight changes (its version counter moves on every in-place update, e.g. an
    optimizer step)."""
    key = (wg._version, wg.data_ptr())
    ent = getattr(wg, "_hm_wg_t", None)
    if ent is None or ent[0] != key:
        ent = (key, ops.transpose_bf16(wg.detach()))
        wg._hm_wg_t = ent
    return ent[1]


class _MoEFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, wg, w_ug, w_down, k, max_ctas):
        # idx is an output without a gradient: do not let autograd materialise a zero int32
        # gradient for it (an eager fill kernel per backward)
        ctx.set_materialize_grads(False)
        r = ops.router_topk(x, wg, k)
        x_perm, row_src, row_of = ops.dispatch_permute(x, r)
        y_perm, h, act = ops.grouped_ffn_fwd(x_perm, r.offsets, w_ug, w_down, max_ctas)
        y = ops.combine(y_perm, row_of, r.w)
        ctx.save_for_backward(x, wg, w_ug, w_down, x_perm, row_of, y_perm, h, act)
        ctx.routing = r
        ctx.max_ctas = max_ctas
        ctx.wg_obj = wg  # the caller's router weight object: key of the cached Wg^T
        ctx.mark_non_differentiable(r.idx)
        return y, r.idx

    @staticmethod
    def backward(ctx, dy, _didx):
        x, wg, w_ug, w_down, x_perm, row_of, y_perm, h, act = ctx.saved_tensors
        r = ctx.routing
        if dy is None:  # y did not reach the loss
            return None, None, None, None, None, None
        dy = dy.contiguous()
        dy_perm, dw = ops.combine_bwd(dy, y_perm, row_of, r.w)
        dx_perm, dw_ug, dw_down = ops.grouped_ffn_bwd(
            dy_perm, x_perm, h, act, r.offsets, w_ug, w_down, ctx.max_ctas
        )
        wg_t = router_weight_t(ctx.wg_obj)
        dx, _dlogit, dwg = ops.router_bwd(dx_perm, row_of, r, dw, x_perm, wg_t, want_dwg=True, x=x)
        return dx, dwg, dw_ug, dw_down, None, None


def moe_forward(x, wg, w_ug, w_down, k: int, max_ctas: int = 0):
    """Functional MoE layer over token rows x [T,d] (made contiguous if it is a strided view):
    returns (y [T,d], idx [T,k])."""
    return _MoEFunction.apply(x.contiguous(), wg, w_ug, w_down, k, max_ctas)


class MoELayer(torch.nn.Module):
    """Router + E SwiGLU experts. Parameters are bf16 on the current CUDA device.

    w_ug holds gate and up projections interleaved in 128-row blocks ([E, 2f, d],
    see ``ops.interleave_gate_up``); w_down is [E, d, f]; wg is [d, E].
    ``max_ctas`` caps the grouped-GEMM grid (per-rank capacity weight, BASELINE C5).
    """

    def __init__(self, d: int, f: int, E: int, k: int, max_ctas: int = 0, device="cuda",
                 dtype=torch.bfloat16):
        super().__init__()
        self.d, self.f, self.E, self.k, self.max_ctas = d, f, E, k, max_ctas
        self.wg = torch.nn.Parameter(torch.empty((d, E), device=device, dtype=dtype))
        self.w_ug = torch.nn.Parameter(torch.empty((E, 2 * f, d), device=device, dtype=dtype))
        self.w_down = torch.nn.Parameter(torch.empty((E, d, f), device=device, dtype=dtype))

    @torch.no_grad()
    def load(self, wg, w_gate, w_up, w_down):
        self.wg.copy_(wg)
        self.w_ug.copy_(ops.interleave_gate_up(w_gate, w_up))
        self.w_down.copy_(w_down)
        return self

    def forward(self, x):
        """x [..., d] (any leading shape, e.g. [batch, seq, d]) -> y of the same shape."""
        y, _ = moe_forward(x.reshape(-1, self.d), self.wg, self.w_ug, self.w_down, self.k, self.max_ctas)
        return y.view(x.shape)
