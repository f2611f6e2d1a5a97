"""CPU oracle for the HeterMoE expert-layer tensor path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module, and only as the checker or the timed CPU
baseline; the product path (``paper_2504_03871_b200``) never calls it.

Parity status — "parity unpinned" for the tensor operators. The reference
(``/root/reference/pkg``, zpsim) contains NO router / permute / expert FFN / combine code: each
is an opaque duration (``src/zpsim/costmodel.py:28-47``, ``taskgraph.py:220-246``) and the spec
excludes real GPU execution (``SPEC.md:8``). The semantics restated here follow the paper text:

* gate / top-k / weighted sum ............ ``PAPER.md:110`` (and ``:358`` for the two-branch bwd)
* dispatch to expert owners, combine back  ``PAPER.md:112,356``
* Mixtral-style SwiGLU experts, top-2 ..... ``PAPER.md:401-421,438``

and the conventions SURVEY §8(c) fixes: ties -> lower expert id, w = softmax over the k
selected logits, dropless and padding-free, permutation stable by (expert, token).
The only reference-pinned quantities at this boundary are aggregate token counts
(``costmodel.py:59-79`` B, ``taskgraph.py:560-575`` conservation), checked in
``tests/test_oracle.py``.

Router logits use the SAME fixed fp32 summation order as the CUDA kernel
(``paper_2504_03871_b200/csrc/moe_kernels.cuh``): per 256-wide block j, lane L of 32 accumulates
i = 256*j + 8*L + q (q = 0..7) with single-rounding multiply-adds (bf16 x bf16 products are
exact in fp32), an xor butterfly over lanes with offsets 16, 8, 4, 2, 1 gives the block
partial, and the block partials are added in block order.
Everything that derives from the logits (indices, counts, offsets, row maps) is therefore
bit-exact; floating outputs are compared with the tolerances written in the tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

BLOCK_F = 128


def bf16_round(a: torch.Tensor) -> torch.Tensor:
    """Round to bf16 and back to fp32 (what the GPU sees)."""
    return a.to(torch.bfloat16).to(torch.float32)


# ---------------------------------------------------------------------------------------------
# router


def router_logits(x: np.ndarray, wg: np.ndarray) -> np.ndarray:
    """Fixed-order fp32 logits. x [T,d] and wg [d,E] hold bf16-representable float32 values.

    Blocked order (the CUDA kernel's, ``csrc/moe_kernels.cuh``): d splits into blocks of 256;
    inside block j lane L accumulates i = 256*j + 8*L + q for q = 0..7 from 0 with one rounding
    per step, the 32 lanes are combined by an xor butterfly (16, 8, 4, 2, 1) into the block
    partial P_j, and the logit is ((P_0 + P_1) + P_2) + ... in block order."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    wg = np.ascontiguousarray(wg, dtype=np.float32)
    T, d = x.shape
    E = wg.shape[1]
    assert d % 256 == 0, "router order is defined for d % 256 == 0"
    nj = d // 256
    xr = x.reshape(T, nj, 32, 8)
    wr = wg.reshape(nj, 32, 8, E)
    acc = np.zeros((T, nj, 32, E), dtype=np.float32)
    for q in range(8):
        prod = xr[:, :, :, q, None] * wr[None, :, :, q, :]  # exact in fp32
        acc = acc + prod  # one rounding == fused multiply-add
    lanes = np.arange(32)
    for off in (16, 8, 4, 2, 1):
        acc = acc + acc[:, :, lanes ^ off, :]
    part = acc[:, :, 0, :]
    out = part[:, 0, :].copy()
    for j in range(1, nj):
        out = out + part[:, j, :]
    return out


_CLIB = None


def _clib():
    """oracle/librouter_ref.so (C restatement, built by `make -C oracle`), or None."""
    global _CLIB
    if _CLIB is None:
        import ctypes
        import os

        p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "librouter_ref.so")
        if os.path.exists(p):
            lib = ctypes.CDLL(p)
            P, I = ctypes.c_void_p, ctypes.c_int
            lib.hm_ref_router_logits.argtypes = [P, P, I, I, I, P]
            lib.hm_ref_topk_softmax.argtypes = [P, I, I, I, P, P]
            lib.hm_ref_permutation.argtypes = [P, I, I, I, P, P, P, P]
            _CLIB = lib
        else:
            _CLIB = False
    return _CLIB or None


def router_logits_c(x_bf16: torch.Tensor, wg_bf16: torch.Tensor) -> np.ndarray:
    """Same fixed-order logits as ``router_logits`` from the C restatement (fast, any size)."""
    lib = _clib()
    if lib is None:
        return router_logits(x_bf16.float().numpy(), wg_bf16.float().numpy())
    x = x_bf16.contiguous().view(torch.int16).numpy()
    w = wg_bf16.contiguous().view(torch.int16).numpy()
    T, d = x.shape
    E = w.shape[1]
    out = np.empty((T, E), dtype=np.float32)
    lib.hm_ref_router_logits(x.ctypes.data, w.ctypes.data, T, d, E, out.ctypes.data)
    return out


def route_c(x_bf16: torch.Tensor, wg_bf16: torch.Tensor, k: int, bias=None) -> "RoutingRef":
    """``route`` with the C restatement doing the heavy loops (for full-size parity checks)."""
    logits = router_logits_c(x_bf16, wg_bf16)
    if bias is not None:
        logits = (logits + np.asarray(bias, dtype=np.float32)[None, :]).astype(np.float32)
    lib = _clib()
    T, E = logits.shape
    if lib is None:
        idx, w = topk_softmax(logits, k)
        counts, offsets = counts_offsets(idx, E)
        row_src, row_of = permutation(idx, E)
        return RoutingRef(logits, idx, w, counts, offsets, row_src, row_of)
    idx = np.empty((T, k), dtype=np.int32)
    w = np.empty((T, k), dtype=np.float32)
    lib.hm_ref_topk_softmax(logits.ctypes.data, T, E, k, idx.ctypes.data, w.ctypes.data)
    counts = np.empty(E, dtype=np.int32)
    offsets = np.empty(E + 1, dtype=np.int32)
    row_src = np.empty(T * k, dtype=np.int32)
    row_of = np.empty((T, k), dtype=np.int32)
    lib.hm_ref_permutation(idx.ctypes.data, T, k, E, counts.ctypes.data, offsets.ctypes.data,
                           row_src.ctypes.data, row_of.ctypes.data)
    return RoutingRef(logits, idx, w, counts, offsets, row_src, row_of)


def topk_softmax(logits: np.ndarray, k: int):
    """Top-k with ties -> lower expert id; w = softmax over the selected logits (fp32).

    Non-finite logits follow one total order, (isnan, -logit, expert id): every number (-inf
    included) ranks before every NaN, equal numbers and NaNs go to the lower id, and each
    expert is selected at most once, so the k indices of a row are always distinct (an all-NaN
    row selects experts 0..k-1 and gets NaN weights; an all -inf row gets NaN weights from
    exp(-inf - -inf)). numpy's lexsort already sorts NaN last; ``router_ref.c`` states the same
    comparator explicitly, and the CUDA kernels reach it by marking selected experts NaN."""
    T, E = logits.shape
    order = np.lexsort((np.broadcast_to(np.arange(E), (T, E)), -logits), axis=-1)
    idx = order[:, :k].astype(np.int32)
    sel = np.take_along_axis(logits, idx, axis=1).astype(np.float32)
    with np.errstate(invalid="ignore", over="ignore"):
        ex = np.exp((sel - sel[:, :1]).astype(np.float32)).astype(np.float32)
        s = np.zeros((T,), dtype=np.float32)
        for j in range(k):
            s = (s + ex[:, j]).astype(np.float32)
        w = (ex / s[:, None]).astype(np.float32)
    return idx, w


def topk_softmax_c(logits: np.ndarray, k: int):
    """``topk_softmax`` through the C restatement (the numpy version when it is not built)."""
    lib = _clib()
    logits = np.ascontiguousarray(logits, dtype=np.float32)
    if lib is None:
        return topk_softmax(logits, k)
    T, E = logits.shape
    idx = np.empty((T, k), dtype=np.int32)
    w = np.empty((T, k), dtype=np.float32)
    lib.hm_ref_topk_softmax(logits.ctypes.data, T, E, k, idx.ctypes.data, w.ctypes.data)
    return idx, w


def counts_offsets(idx: np.ndarray, E: int):
    counts = np.bincount(idx.reshape(-1), minlength=E).astype(np.int32)
    offsets = np.zeros(E + 1, dtype=np.int32)
    offsets[1:] = np.cumsum(counts)
    return counts, offsets


def permutation(idx: np.ndarray, E: int):
    """Stable (expert, token) order. Returns row_src [T*k] and row_of [T,k]."""
    T, k = idx.shape
    flat_e = idx.reshape(-1).astype(np.int64)
    flat_t = np.repeat(np.arange(T), k)
    order = np.lexsort((flat_t, flat_e))  # primary expert, secondary token
    row_src = flat_t[order].astype(np.int32)
    row_of = np.empty(T * k, dtype=np.int32)
    row_of[order] = np.arange(T * k, dtype=np.int32)
    return row_src, row_of.reshape(T, k)


@dataclass
class RoutingRef:
    logits: np.ndarray
    idx: np.ndarray
    w: np.ndarray
    counts: np.ndarray
    offsets: np.ndarray
    row_src: np.ndarray
    row_of: np.ndarray


def route(x: np.ndarray, wg: np.ndarray, k: int, bias=None) -> RoutingRef:
    with np.errstate(invalid="ignore", over="ignore"):  # non-finite rows follow IEEE, as on the GPU
        logits = router_logits(x, wg)
        if bias is not None:
            logits = (logits + np.asarray(bias, dtype=np.float32)[None, :]).astype(np.float32)
    idx, w = topk_softmax(logits, k)
    E = wg.shape[1]
    counts, offsets = counts_offsets(idx, E)
    row_src, row_of = permutation(idx, E)
    return RoutingRef(logits, idx, w, counts, offsets, row_src, row_of)


# ---------------------------------------------------------------------------------------------
# expert FFN / combine in fp32 (torch CPU autograd for the backward)


def split_gate_up(w_ug: torch.Tensor, block: int = BLOCK_F):
    E, two_f, d = w_ug.shape
    f = two_f // 2
    v = w_ug.reshape(E, f // block, 2, block, d)
    return v[:, :, 0].reshape(E, f, d), v[:, :, 1].reshape(E, f, d)


def expert_ffn(x_perm: torch.Tensor, offsets, w_gate, w_up, w_down) -> torch.Tensor:
    """Per expert e: Y = (silu(X Wg^T) * (X Wu^T)) Wd^T over rows [offsets[e], offsets[e+1])."""
    outs = []
    for e in range(len(w_gate)):
        a, b = int(offsets[e]), int(offsets[e + 1])
        xe = x_perm[a:b]
        g = xe @ w_gate[e].t()
        u = xe @ w_up[e].t()
        outs.append((torch.nn.functional.silu(g) * u) @ w_down[e].t())
    return torch.cat(outs, 0) if outs else x_perm.new_zeros((0, w_down.shape[1]))


def moe_layer(x, wg, w_ug, w_down, k: int, dy=None, routing: RoutingRef | None = None):
    """Full MoE layer forward (+ backward if dy is given) in fp32 on the CPU.

    Inputs are fp32 tensors holding bf16-representable values. Returns a dict with the
    routing (numpy, bit-exact reference) and y / dx / dwg / dw_ug / dw_down (fp32 torch).
    """
    x = x.detach().float().cpu()
    wg = wg.detach().float().cpu()
    w_gate, w_up = split_gate_up(w_ug.detach().float().cpu())
    w_down = w_down.detach().float().cpu()
    r = routing or route(x.numpy(), wg.numpy(), k)
    T = x.shape[0]

    xg = x.clone().requires_grad_(dy is not None)
    wgg = wg.clone().requires_grad_(dy is not None)
    # one leaf per expert (indexing a stacked leaf would materialise a full-size zero gradient
    # per expert in the backward)
    rg = dy is not None
    wgt = [w_gate[e].clone().requires_grad_(rg) for e in range(w_gate.shape[0])]
    wut = [w_up[e].clone().requires_grad_(rg) for e in range(w_up.shape[0])]
    wdt = [w_down[e].clone().requires_grad_(rg) for e in range(w_down.shape[0])]

    logits = xg @ wgg  # values differ from the fixed-order logits only by rounding
    idx_t = torch.from_numpy(r.idx.astype(np.int64))
    sel = torch.gather(logits, 1, idx_t)
    w = torch.softmax(sel, dim=1)
    row_src = torch.from_numpy(r.row_src.astype(np.int64))
    x_perm = xg[row_src]
    y_perm = expert_ffn(x_perm, r.offsets, wgt, wut, wdt)
    row_of = torch.from_numpy(r.row_of.astype(np.int64))
    y = (y_perm[row_of.reshape(-1)].reshape(T, k, -1) * w[:, :, None]).sum(1)
    out = {"routing": r, "y": y.detach(), "w": w.detach()}
    if dy is not None:
        y.backward(dy.detach().float().cpu())
        stack = lambda ws: torch.stack([w.grad if w.grad is not None else torch.zeros_like(w) for w in ws])  # noqa: E731
        out.update(dx=xg.grad, dwg=wgg.grad, dw_gate=stack(wgt), dw_up=stack(wut), dw_down=stack(wdt))
    return out


class CpuLayer:
    """The same fp32 CPU layer as ``moe_layer`` with its parameters converted ONCE (fp32 master
    copies with gradients), for timing the CPU path per step (bench.py's ``cpu_baseline`` and
    ``--impl reference`` arms): each ``step`` routes (fixed-order oracle), runs the forward and
    the backward, and leaves the gradients in the parameters."""

    def __init__(self, wg, w_ug, w_down, k: int):
        self.k = k
        self.wg = wg.detach().float().cpu().clone().requires_grad_()
        g, u = split_gate_up(w_ug.detach().float().cpu())
        # one leaf per expert: indexing a stacked [E, ...] leaf would make autograd materialise
        # a full-size zero gradient per expert (SelectBackward)
        self.w_gate = [g[e].contiguous().requires_grad_() for e in range(g.shape[0])]
        self.w_up = [u[e].contiguous().requires_grad_() for e in range(u.shape[0])]
        wd = w_down.detach().float().cpu()
        self.w_down = [wd[e].contiguous().requires_grad_() for e in range(wd.shape[0])]

    def params(self):
        return [self.wg] + self.w_gate + self.w_up + self.w_down

    def step(self, x, dy):
        for p in self.params():
            p.grad = None
        x = x.detach().float().cpu()
        r = route(x.numpy(), self.wg.detach().numpy(), self.k)
        T = x.shape[0]
        xg = x.requires_grad_()
        logits = xg @ self.wg
        w = torch.softmax(torch.gather(logits, 1, torch.from_numpy(r.idx.astype(np.int64))), dim=1)
        x_perm = xg[torch.from_numpy(r.row_src.astype(np.int64))]
        y_perm = expert_ffn(x_perm, r.offsets, self.w_gate, self.w_up, self.w_down)
        row_of = torch.from_numpy(r.row_of.astype(np.int64))
        y = (y_perm[row_of.reshape(-1)].reshape(T, self.k, -1) * w[:, :, None]).sum(1)
        y.backward(dy.detach().float().cpu())
        return y.detach()


def rel_err(a: torch.Tensor, b: torch.Tensor) -> float:
    """Relative Frobenius error ||a-b|| / ||b||."""
    a = a.detach().float().cpu()
    b = b.detach().float().cpu()
    den = torch.linalg.vector_norm(b).item()
    return torch.linalg.vector_norm(a - b).item() / (den if den > 0 else 1.0)
