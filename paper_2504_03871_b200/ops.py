"""Tensor-level operators of the expert-layer hot path (router, dispatch, expert FFN, combine).

Each function wraps one C-ABI entry point of ``libhetermoe_kernels.so`` and runs it on the
current torch CUDA stream. There is no CPU fallback: inputs must be CUDA tensors and the
native library must be present (``_native.NativeLibraryError`` otherwise).

Reference anchors: the reference folds all of these into opaque task durations
(router/permute/combine -> ATTN_F, ``/root/reference/pkg/src/zpsim/taskgraph.py:220-246``;
expert FFN -> EXP_F, ``costmodel.py:28-37``); their semantics come from the paper
(``PAPER.md:110,112,356,358``) and are pinned by ``oracle/moe_oracle.py``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import torch

from . import _native

BLOCK_F = 128  # gate/up interleave block of the fused W_ug layout

# number of native kernel launches issued through this module (bench.py's gpu_launches);
# (a lock, in case several host threads issue native ops)
LAUNCHES = [0]
_LAUNCH_LOCK = threading.Lock()


def _count(n: int) -> None:
    with _LAUNCH_LOCK:
        LAUNCHES[0] += n


class KernelTimer:
    """Records CUDA events around every native call on the launching stream (bench.py uses it
    over the timed region to get per-kernel device durations)."""

    def __init__(self):
        self.events = {}  # name -> list of (start, end) events

    def begin(self, name: str):
        s = torch.cuda.Event(enable_timing=True)
        s.record()
        return name, s

    def end(self, tok) -> None:
        name, s = tok
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.events.setdefault(name, []).append((s, e))

    def summary(self) -> dict:
        """name -> (launch count, total ms); call after synchronising."""
        return {n: (len(v), sum(a.elapsed_time(b) for a, b in v)) for n, v in self.events.items()}


_TIMER: list = [None]


def set_timer(timer: "KernelTimer | None") -> None:
    _TIMER[0] = timer


def _begin(name: str):
    t = _TIMER[0]
    return t.begin(name) if t is not None else None


def _end(tok) -> None:
    if tok is not None:
        _TIMER[0].end(tok)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _require_cuda(*ts: torch.Tensor) -> None:
    dev = None
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("hetermoe ops need contiguous CUDA tensors (no CPU fallback)")
        if dev is None:
            dev = torch.cuda.current_device()
        if t.device.index != dev:
            raise ValueError(f"hetermoe ops run on the current CUDA device (cuda:{dev}); got a tensor "
                             f"on {t.device} (use torch.cuda.device(...) around the call)")


def _require_dtype(**named) -> None:
    """name=(tensor or None, dtype): the kernels read raw bytes, so a wrong dtype is an error."""
    for name, (t, dt) in named.items():
        if t is not None and t.dtype != dt:
            raise TypeError(f"hetermoe: {name} must be {dt}, got {t.dtype}")


@dataclass
class Routing:
    """Result of the router: everything dispatch / combine need."""

    idx: torch.Tensor  # [T, k] int32 expert ids, descending logit
    w: torch.Tensor  # [T, k] fp32 gate weights (softmax over the k)
    logits: torch.Tensor  # [T, E] fp32
    counts: torch.Tensor  # [E] int32 tokens per expert
    offsets: torch.Tensor  # [E+1] int32 exclusive prefix sum of counts
    chunk_base: torch.Tensor  # [nchunk, E] int32 per-chunk row bases


def router_topk(x: torch.Tensor, wg: torch.Tensor, k: int, bias: torch.Tensor | None = None) -> Routing:
    """K1: fixed-order fp32 logits (+ optional per-expert fp32 bias), top-k (ties -> lower id),
    softmax over the k, per-expert histogram and offsets."""
    _require_cuda(x, wg, bias)
    _require_dtype(x=(x, torch.bfloat16), wg=(wg, torch.bfloat16), bias=(bias, torch.float32))
    lib = _native.load()
    T, d = x.shape
    E = wg.shape[1]
    dev = x.device
    idx = torch.empty((T, k), dtype=torch.int32, device=dev)
    w = torch.empty((T, k), dtype=torch.float32, device=dev)
    logits = torch.empty((T, E), dtype=torch.float32, device=dev)
    counts = torch.empty((E,), dtype=torch.int32, device=dev)
    offsets = torch.empty((E + 1,), dtype=torch.int32, device=dev)
    nce = lib.hm_router_chunk_elems(T, E)
    chunk_base = torch.empty((max(nce, 1),), dtype=torch.int32, device=dev)
    _tk = _begin("router_topk")
    rc = lib.hm_router_topk(
        _ptr(x), _ptr(wg), _ptr(bias), T, d, E, k, _ptr(idx), _ptr(w), _ptr(logits), _ptr(counts),
        _ptr(offsets), _ptr(chunk_base), _stream(),
    )
    _end(_tk)
    _native.check(rc, "hm_router_topk")
    _count(lib.hm_router_launches(T, d, E))
    return Routing(idx, w, logits, counts, offsets, chunk_base)


def dispatch_permute(x: torch.Tensor, r: Routing, out: torch.Tensor | None = None):
    """K2: x[T,d] -> (x_perm[T*k,d] grouped by expert, row_src[T*k], row_of[T,k])."""
    _require_cuda(x)
    _require_dtype(x=(x, torch.bfloat16))
    T, d = x.shape
    k = r.idx.shape[1]
    E = r.counts.shape[0]
    dev = x.device
    x_perm = out if out is not None else torch.empty((T * k, d), dtype=x.dtype, device=dev)
    row_src = torch.empty((T * k,), dtype=torch.int32, device=dev)
    row_of = torch.empty((T, k), dtype=torch.int32, device=dev)
    _tk = _begin("dispatch_permute")
    rc = _native.load().hm_dispatch_permute(
        _ptr(x), _ptr(r.idx), _ptr(r.chunk_base), T, d, E, k, _ptr(x_perm), _ptr(row_src),
        _ptr(row_of), _stream(),
    )
    _end(_tk)
    _native.check(rc, "hm_dispatch_permute")
    _count(1)
    return x_perm, row_src, row_of


def unpermute_sum(dx_perm: torch.Tensor, row_of: torch.Tensor) -> torch.Tensor:
    _require_cuda(dx_perm, row_of)
    _require_dtype(dx_perm=(dx_perm, torch.bfloat16), row_of=(row_of, torch.int32))
    T, k = row_of.shape
    d = dx_perm.shape[1]
    dx = torch.empty((T, d), dtype=dx_perm.dtype, device=dx_perm.device)
    _tk = _begin("unpermute_sum")
    rc = _native.load().hm_unpermute_sum(_ptr(dx_perm), _ptr(row_of), T, d, k, _ptr(dx), _stream())
    _end(_tk)
    _native.check(rc, "hm_unpermute_sum")
    _count(1)
    return dx


def combine(y_perm: torch.Tensor, row_of: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """K4: y[t] = sum_s w[t,s] * y_perm[row_of[t,s]]."""
    _require_cuda(y_perm, row_of, w)
    _require_dtype(y_perm=(y_perm, torch.bfloat16), row_of=(row_of, torch.int32), w=(w, torch.float32))
    T, k = row_of.shape
    d = y_perm.shape[1]
    y = torch.empty((T, d), dtype=y_perm.dtype, device=y_perm.device)
    _tk = _begin("combine")
    rc = _native.load().hm_combine(_ptr(y_perm), _ptr(row_of), _ptr(w), T, d, k, _ptr(y), _stream())
    _end(_tk)
    _native.check(rc, "hm_combine")
    _count(1)
    return y


def combine_bwd(dy: torch.Tensor, y_perm: torch.Tensor, row_of: torch.Tensor, w: torch.Tensor):
    _require_cuda(dy, y_perm, row_of, w)
    _require_dtype(dy=(dy, torch.bfloat16), y_perm=(y_perm, torch.bfloat16), row_of=(row_of, torch.int32),
                   w=(w, torch.float32))
    T, k = row_of.shape
    d = dy.shape[1]
    dy_perm = torch.empty_like(y_perm)
    dw = torch.empty((T, k), dtype=torch.float32, device=dy.device)
    _tk = _begin("combine_bwd")
    rc = _native.load().hm_combine_bwd(
        _ptr(dy), _ptr(y_perm), _ptr(row_of), _ptr(w), T, d, k, _ptr(dy_perm), _ptr(dw), _stream()
    )
    _end(_tk)
    _native.check(rc, "hm_combine_bwd")
    _count(1)
    return dy_perm, dw


def transpose_bf16(a: torch.Tensor) -> torch.Tensor:
    _require_cuda(a)
    R, C = a.shape
    out = torch.empty((C, R), dtype=a.dtype, device=a.device)
    _tk = _begin("transpose_bf16")
    rc = _native.load().hm_transpose_bf16(_ptr(a), R, C, _ptr(out), _stream())
    _end(_tk)
    _native.check(rc, "hm_transpose_bf16")
    _count(1)
    return out


def router_bwd(dx_perm, row_of, r: Routing, dw, x_perm, wg_t, want_dwg: bool = True, x=None):
    """dx = unpermute_sum(dx_perm) + dlogit . Wg^T ; dWg = x^T . dlogit_dense (E <= 8: from the token
    rows x when given, streamed; else from the routed copies in x_perm)."""
    _require_cuda(dx_perm, row_of, dw, x_perm, wg_t, x)
    lib = _native.load()
    T, k = row_of.shape
    d = x_perm.shape[1]
    E = wg_t.shape[0]
    dev = x_perm.device
    dx = torch.empty((T, d), dtype=x_perm.dtype, device=dev)
    dlogit = torch.empty((T, k), dtype=torch.float32, device=dev)
    dwg = part = None
    if want_dwg:
        dwg = torch.empty((d, E), dtype=x_perm.dtype, device=dev)
        part = torch.empty((lib.hm_router_bwd_part_elems(T, d, E, k),), dtype=torch.float32, device=dev)
    _tk = _begin("router_bwd")
    rc = lib.hm_router_bwd(
        _ptr(dx_perm), _ptr(row_of), _ptr(r.idx), _ptr(r.w), _ptr(dw), _ptr(x), _ptr(x_perm), _ptr(r.offsets),
        _ptr(wg_t), T, d, E, k, _ptr(dx), _ptr(dlogit), _ptr(dwg), _ptr(part), _stream(),
    )
    _end(_tk)
    _native.check(rc, "hm_router_bwd")
    _count(3 if want_dwg else 1)
    return dx, dlogit, dwg


def grouped_gemm(mode: int, a, b, seg_offsets, E: int, rows: int, M: int, N: int, K: int, out,
                 ldo: int, out2=None, ldo2: int = 0, aux=None, ld_aux: int = 0,
                 max_ctas: int = 0, name: str = "grouped_gemm") -> None:
    """One launch of the tcgen05 grouped GEMM (modes: _native.GEMM_*). The WGRAD modes get a
    small device workspace for their per-expert TMA views."""
    lib = _native.load()
    ws = None
    nbytes = lib.hm_grouped_gemm_workspace_bytes(mode, E)
    if nbytes:
        ws = torch.empty((nbytes + 128,), dtype=torch.uint8, device=a.device)
        off = (-ws.data_ptr()) % 128
        ws = ws[off:off + nbytes]
    _tk = _begin(name)
    rc = lib.hm_grouped_gemm(
        mode, _ptr(a), _ptr(b), _ptr(seg_offsets), E, rows, M, N, K, _ptr(out), ldo, _ptr(out2),
        ldo2, _ptr(aux), ld_aux, _ptr(ws), max_ctas, _stream(),
    )
    _end(_tk)
    _native.check(rc, "hm_grouped_gemm")
    _count(2 if nbytes else 1)  # the weight-gradient modes first build their per-expert TMA views


def grouped_ffn_fwd(x_perm, seg_offsets, w_ug, w_d, max_ctas: int = 0):
    """K3 forward (same math as hm_grouped_ffn_fwd, one launch per GEMM so each is timed):
    h = x_perm . w_ug[e]^T (gate|up), act = silu(gate)*up, y_perm = act . w_d[e]^T.
    Returns (y_perm, h, act). w_ug [E,2f,d] interleaved, w_d [E,d,f]."""
    _require_cuda(x_perm, seg_offsets, w_ug, w_d)
    _require_dtype(x_perm=(x_perm, torch.bfloat16), seg_offsets=(seg_offsets, torch.int32),
                   w_ug=(w_ug, torch.bfloat16), w_d=(w_d, torch.bfloat16))
    rows, d = x_perm.shape
    E, two_f, _ = w_ug.shape
    f = two_f // 2
    dev = x_perm.device
    h = torch.empty((rows, 2 * f), dtype=x_perm.dtype, device=dev)
    act = torch.empty((rows, f), dtype=x_perm.dtype, device=dev)
    y_perm = torch.empty((rows, d), dtype=x_perm.dtype, device=dev)
    grouped_gemm(_native.GEMM_FWD_UPGATE, x_perm, w_ug, seg_offsets, E, rows, 0, 2 * f, d, act, f,
                 out2=h, ldo2=2 * f, max_ctas=max_ctas, name="gemm_fwd_upgate")
    grouped_gemm(_native.GEMM_FWD_DOWN, act, w_d, seg_offsets, E, rows, 0, d, f, y_perm, d,
                 max_ctas=max_ctas, name="gemm_fwd_down")
    return y_perm, h, act


def grouped_ffn_bwd(dy_perm, x_perm, h, act, seg_offsets, w_ug, w_d, max_ctas: int = 0):
    """K3 backward: dh = SwiGLU'(dy_perm . w_d[e]); dx_perm = dh . w_ug[e];
    dw_ug[e] = dh_e^T . x_e; dw_d[e] = dy_e^T . act_e. Returns (dx_perm, dw_ug, dw_d)."""
    _require_cuda(dy_perm, x_perm, h, act, seg_offsets, w_ug, w_d)
    _require_dtype(dy_perm=(dy_perm, torch.bfloat16), x_perm=(x_perm, torch.bfloat16), h=(h, torch.bfloat16),
                   act=(act, torch.bfloat16), seg_offsets=(seg_offsets, torch.int32),
                   w_ug=(w_ug, torch.bfloat16), w_d=(w_d, torch.bfloat16))
    rows, d = x_perm.shape
    E, two_f, _ = w_ug.shape
    f = two_f // 2
    dev = x_perm.device
    dh = torch.empty((rows, 2 * f), dtype=x_perm.dtype, device=dev)
    dx_perm = torch.empty((rows, d), dtype=x_perm.dtype, device=dev)
    dw_ug = torch.empty_like(w_ug)
    dw_d = torch.empty_like(w_d)
    grouped_gemm(_native.GEMM_BWD_DACT, dy_perm, w_d, seg_offsets, E, rows, 0, f, d, dh, 2 * f,
                 aux=h, ld_aux=2 * f, max_ctas=max_ctas, name="gemm_bwd_dact")
    grouped_gemm(_native.GEMM_BWD_DX, dh, w_ug, seg_offsets, E, rows, 0, d, 2 * f, dx_perm, d,
                 max_ctas=max_ctas, name="gemm_bwd_dx")
    grouped_gemm(_native.GEMM_WGRAD, dh, x_perm, seg_offsets, E, rows, 2 * f, d, 0, dw_ug, d,
                 max_ctas=max_ctas, name="gemm_wgrad_ug")
    grouped_gemm(_native.GEMM_WGRAD, dy_perm, act, seg_offsets, E, rows, d, f, 0, dw_d, f,
                 max_ctas=max_ctas, name="gemm_wgrad_down")
    return dx_perm, dw_ug, dw_d


def grouped_ffn_bwd_data(dy_perm, x_perm, h, act, seg_offsets, w_ug, w_d, max_ctas: int = 0):
    """Data-gradient half of the FFN backward: dh = SwiGLU'(dy . w_d[e]), dx = dh . w_ug[e].
    Returns (dx_perm, dh); the weight gradients are formed later by grouped_wgrad_multi."""
    _require_cuda(dy_perm, x_perm, h, act, seg_offsets, w_ug, w_d)
    _require_dtype(dy_perm=(dy_perm, torch.bfloat16), x_perm=(x_perm, torch.bfloat16), h=(h, torch.bfloat16),
                   act=(act, torch.bfloat16), seg_offsets=(seg_offsets, torch.int32),
                   w_ug=(w_ug, torch.bfloat16), w_d=(w_d, torch.bfloat16))
    rows, d = x_perm.shape
    E, two_f, _ = w_ug.shape
    f = two_f // 2
    dh = torch.empty((rows, 2 * f), dtype=x_perm.dtype, device=x_perm.device)
    dx_perm = torch.empty((rows, d), dtype=x_perm.dtype, device=x_perm.device)
    grouped_gemm(_native.GEMM_BWD_DACT, dy_perm, w_d, seg_offsets, E, rows, 0, f, d, dh, 2 * f,
                 aux=h, ld_aux=2 * f, max_ctas=max_ctas, name="gemm_bwd_dact")
    grouped_gemm(_native.GEMM_BWD_DX, dh, w_ug, seg_offsets, E, rows, 0, d, 2 * f, dx_perm, d,
                 max_ctas=max_ctas, name="gemm_bwd_dx")
    return dx_perm, dh


def grouped_wgrad_multi(a_list, b_list, seg_multi, out, accumulate: bool = True,
                        max_ctas: int = 0, name: str = "gemm_wgrad_multi") -> None:
    """out[e] (+)= sum_j a_list[j][seg_j(e)]^T . b_list[j][seg_j(e)] in ONE grouped GEMM whose K
    loop runs over every segment (micro-batch). seg_multi: int32 [R, E+1] on the device."""
    lib = _native.load()
    R = len(a_list)
    if not accumulate and (R > 16 or out.dtype != torch.bfloat16):
        raise ValueError("non-accumulating grouped_wgrad_multi needs bf16 out and at most 16 segments")
    if accumulate and out.dtype != torch.float32:
        raise ValueError("accumulating grouped_wgrad_multi needs an fp32 out")
    E = seg_multi.shape[1] - 1
    M = a_list[0].shape[1]
    N = b_list[0].shape[1]
    dev = a_list[0].device
    for j0 in range(0, R, 16):
        a = a_list[j0:j0 + 16]
        b = b_list[j0:j0 + 16]
        r = len(a)
        nbytes = lib.hm_grouped_wgrad_multi_workspace_bytes(E, r)
        ws = torch.empty((nbytes + 128,), dtype=torch.uint8, device=dev)
        off = (-ws.data_ptr()) % 128
        ws = ws[off:off + nbytes]
        ap = (ctypes.c_void_p * r)(*[t.data_ptr() for t in a])
        bp = (ctypes.c_void_p * r)(*[t.data_ptr() for t in b])
        rows = (ctypes.c_int * r)(*[t.shape[0] for t in a])
        seg = seg_multi[j0:j0 + r].contiguous()
        acc = 1 if (accumulate or j0 > 0) else 0
        _tk = _begin(name)
        rc = lib.hm_grouped_wgrad_multi(acc, ap, bp, rows, _ptr(seg), r, E, M, N, _ptr(out), N,
                                        _ptr(ws), max_ctas, _stream())
        _end(_tk)
        _native.check(rc, "hm_grouped_wgrad_multi")
        _count(2)


def grouped_ffn_bwd_acc(dy_perm, x_perm, h, act, seg_offsets, w_ug, w_d, gw_ug, gw_d,
                        max_ctas: int = 0):
    """Backward with fp32 weight-gradient ACCUMULATION (gw_ug [E,2f,d], gw_d [E,d,f] fp32 +=),
    used when gradients accumulate over micro-batches. Returns dx_perm."""
    _require_cuda(dy_perm, x_perm, h, act, seg_offsets, w_ug, w_d, gw_ug, gw_d)
    rows, d = x_perm.shape
    E, two_f, _ = w_ug.shape
    f = two_f // 2
    dev = x_perm.device
    dh = torch.empty((rows, 2 * f), dtype=x_perm.dtype, device=dev)
    dx_perm = torch.empty((rows, d), dtype=x_perm.dtype, device=dev)
    grouped_gemm(_native.GEMM_BWD_DACT, dy_perm, w_d, seg_offsets, E, rows, 0, f, d, dh, 2 * f,
                 aux=h, ld_aux=2 * f, max_ctas=max_ctas, name="gemm_bwd_dact")
    grouped_gemm(_native.GEMM_BWD_DX, dh, w_ug, seg_offsets, E, rows, 0, d, 2 * f, dx_perm, d,
                 max_ctas=max_ctas, name="gemm_bwd_dx")
    grouped_gemm(_native.GEMM_WGRAD_ACC, dh, x_perm, seg_offsets, E, rows, 2 * f, d, 0, gw_ug, d,
                 max_ctas=max_ctas, name="gemm_wgrad_ug")
    grouped_gemm(_native.GEMM_WGRAD_ACC, dy_perm, act, seg_offsets, E, rows, d, f, 0, gw_d, f,
                 max_ctas=max_ctas, name="gemm_wgrad_down")
    return dx_perm


# ---------------------------------------------------------------------------------------------
# weight layout helpers (host side, any device)


def interleave_gate_up(w_gate: torch.Tensor, w_up: torch.Tensor, block: int = BLOCK_F) -> torch.Tensor:
    """[E,f,d] gate and up weights -> fused [E,2f,d] with 128-row gate/up blocks alternating."""
    E, f, d = w_gate.shape
    assert f % block == 0
    g = w_gate.reshape(E, f // block, block, d)
    u = w_up.reshape(E, f // block, block, d)
    return torch.stack([g, u], dim=2).reshape(E, 2 * f, d).contiguous()


def split_gate_up(w_ug: torch.Tensor, block: int = BLOCK_F):
    """Inverse of interleave_gate_up."""
    E, two_f, d = w_ug.shape
    f = two_f // 2
    v = w_ug.reshape(E, f // block, 2, block, d)
    return v[:, :, 0].reshape(E, f, d), v[:, :, 1].reshape(E, f, d)


# ---------------------------------------------------------------------------------------------
# NVLink peer-memory transport (fused compute + dispatch / combine; used by executor.P2P)


def dispatch_permute_p2p(x: torch.Tensor, r: Routing, dest_base: torch.Tensor, dest_start: torch.Tensor,
                         keep_local: bool = True):
    """Fused permute + dispatch: each routed row goes to its expert owner's receive buffer
    (dest_base[e] + (dest_start[e] + row - offsets[e]) * d, possibly a peer GPU); optionally also
    to the local permuted buffer. Returns (x_perm or None, row_of)."""
    _require_cuda(x, dest_base, dest_start)
    T, d = x.shape
    k = r.idx.shape[1]
    E = r.counts.shape[0]
    x_perm = torch.empty((T * k, d), dtype=x.dtype, device=x.device) if keep_local else None
    row_of = torch.empty((T, k), dtype=torch.int32, device=x.device)
    _tk = _begin("dispatch_permute_p2p")
    rc = _native.load().hm_dispatch_permute_p2p(
        _ptr(x), _ptr(r.idx), _ptr(r.chunk_base), _ptr(r.offsets), T, d, E, k, _ptr(x_perm), None,
        _ptr(row_of), _ptr(dest_base), _ptr(dest_start), _stream())
    _end(_tk)
    _native.check(rc, "hm_dispatch_permute_p2p")
    _count(1)
    return x_perm, row_of


def combine_bwd_p2p(dy, y_perm, row_of, r: Routing, dest_base, dest_start):
    """Fused combine backward + dispatch of dY rows to the owners; returns dw [T,k] (local)."""
    _require_cuda(dy, y_perm, row_of, dest_base, dest_start)
    T, k = row_of.shape
    d = dy.shape[1]
    dw = torch.empty((T, k), dtype=torch.float32, device=dy.device)
    _tk = _begin("combine_bwd_p2p")
    rc = _native.load().hm_combine_bwd_p2p(
        _ptr(dy), _ptr(y_perm), _ptr(row_of), _ptr(r.idx), _ptr(r.w), _ptr(r.offsets), T, d, k,
        _ptr(dest_base), _ptr(dest_start), _ptr(dw), _stream())
    _end(_tk)
    _native.check(rc, "hm_combine_bwd_p2p")
    _count(1)
    return dw


def _gemm_rows(mode, a, b, seg, E, rows, N, K, out_rows, max_ctas, name):
    _tk = _begin(name)
    rc = _native.load().hm_grouped_gemm_rows(mode, _ptr(a), _ptr(b), _ptr(seg), E, rows, 0, N, K, None,
                                             N, None, 0, None, 0, None, _ptr(out_rows), max_ctas,
                                             _stream())
    _end(_tk)
    _native.check(rc, "hm_grouped_gemm_rows")
    _count(1)


def grouped_ffn_fwd_rows(x_perm, seg_offsets, w_ug, w_d, out_rows, max_ctas: int = 0):
    """Forward whose down-projection epilogue writes output row r to out_rows[r] (the combine
    return fused into the GEMM). Returns (h, act)."""
    _require_cuda(x_perm, seg_offsets, w_ug, w_d, out_rows)
    rows, d = x_perm.shape
    E, two_f, _ = w_ug.shape
    f = two_f // 2
    h = torch.empty((rows, 2 * f), dtype=x_perm.dtype, device=x_perm.device)
    act = torch.empty((rows, f), dtype=x_perm.dtype, device=x_perm.device)
    grouped_gemm(_native.GEMM_FWD_UPGATE, x_perm, w_ug, seg_offsets, E, rows, 0, 2 * f, d, act, f,
                 out2=h, ldo2=2 * f, max_ctas=max_ctas, name="gemm_fwd_upgate")
    _gemm_rows(_native.GEMM_FWD_DOWN, act, w_d, seg_offsets, E, rows, d, f, out_rows, max_ctas,
               "gemm_fwd_down_p2p")
    return h, act


def grouped_ffn_bwd_data_rows(dy_perm, x_perm, h, act, seg_offsets, w_ug, w_d, out_rows, max_ctas: int = 0):
    """Data-gradient backward whose dX epilogue writes row r to out_rows[r]. Returns dh."""
    _require_cuda(dy_perm, x_perm, h, act, seg_offsets, w_ug, w_d, out_rows)
    rows, d = x_perm.shape
    E, two_f, _ = w_ug.shape
    f = two_f // 2
    dh = torch.empty((rows, 2 * f), dtype=x_perm.dtype, device=x_perm.device)
    grouped_gemm(_native.GEMM_BWD_DACT, dy_perm, w_d, seg_offsets, E, rows, 0, f, d, dh, 2 * f,
                 aux=h, ld_aux=2 * f, max_ctas=max_ctas, name="gemm_bwd_dact")
    _gemm_rows(_native.GEMM_BWD_DX, dh, w_ug, seg_offsets, E, rows, d, 2 * f, out_rows, max_ctas,
               "gemm_bwd_dx_p2p")
    return dh


# Device-side receive layout + pool-placed expert activations (executor.ZpP2PExecutor, no host
# read of the routed counts)


def zp_layout(counts_all, M: int, owners, me: int, n_own: int, cap: int, y_base, dx_delta: int,
              row_bytes: int, dest_start, seg, out_rows_y, out_rows_dx, shifts, top, pool_base: int,
              pool_rows: int, err) -> None:
    """hm_zp_layout: from the all-gathered counts [>=M, E] (device), this rank's send table
    dest_start[E] (attention ranks) and, for an owner of n_own experts, its segment table, the
    per-row return addresses and the pool row shifts of its four expert GEMMs."""
    E = owners.shape[0]
    _tk = _begin("zp_layout")
    rc = _native.load().hm_zp_layout(
        _ptr(counts_all), M, E, _ptr(owners), me, n_own, cap, _ptr(y_base), dx_delta, row_bytes,
        _ptr(dest_start), _ptr(seg), _ptr(out_rows_y), _ptr(out_rows_dx), _ptr(shifts), _ptr(top),
        pool_base, pool_rows, _ptr(err), _stream())
    _end(_tk)
    _native.check(rc, "hm_zp_layout")
    _count(1)


def _gemm_shifted(mode, a_ptr: int, b, seg, E, rows, a_rows, N, K, out=None, ldo=0, out2=None, ldo2=0,
                  aux=None, ld_aux=0, out_rows=None, row_shift=None, max_ctas=0, name="grouped_gemm"):
    _tk = _begin(name)
    rc = _native.load().hm_grouped_gemm_shifted(
        mode, a_ptr, _ptr(b), _ptr(seg), E, rows, a_rows, 0, N, K, _ptr(out), ldo if ldo else N, _ptr(out2), ldo2,
        _ptr(aux), ld_aux, None, _ptr(out_rows), _ptr(row_shift), max_ctas, _stream())
    _end(_tk)
    _native.check(rc, "hm_grouped_gemm_shifted")
    _count(1)


def grouped_ffn_fwd_pool(x_slot, seg, w_ug, w_d, h_pool, act_pool, shifts, out_rows, cap: int,
                         max_ctas: int = 0) -> None:
    """Forward over a receive slot (x_slot[:cap], expert segments in seg, device) whose h / act go
    to pool rows at the device-computed base (shifts[0:2]) and whose down projection stores row r
    at out_rows[r] (the combine return), reading act at shifts[2:4]."""
    _require_cuda(x_slot, seg, w_ug, w_d, h_pool, act_pool, shifts, out_rows)
    d = x_slot.shape[1]
    E, two_f, _ = w_ug.shape
    f = two_f // 2
    _gemm_shifted(_native.GEMM_FWD_UPGATE, x_slot.data_ptr(), w_ug, seg, E, cap, cap, 2 * f, d,
                  out=act_pool, ldo=f, out2=h_pool, ldo2=2 * f, row_shift=shifts[0:2], max_ctas=max_ctas,
                  name="gemm_fwd_upgate")
    _gemm_shifted(_native.GEMM_FWD_DOWN, act_pool.data_ptr(), w_d, seg, E, cap, act_pool.shape[0], d, f,
                  out_rows=out_rows, row_shift=shifts[2:4], max_ctas=max_ctas, name="gemm_fwd_down_p2p")


def grouped_ffn_bwd_data_pool(dy_slot, seg, w_ug, w_d, h_pool, dh_ptr: int, dh_rows: int, shifts, out_rows,
                              cap: int, max_ctas: int = 0) -> None:
    """Data-gradient backward over a receive slot: dH (SwiGLU backward, reading h at the pool base)
    goes to the dh buffer at dh_ptr (addressed with the same pool rows, dh_rows of them), and the
    dX GEMM stores row r at out_rows[r]."""
    _require_cuda(dy_slot, seg, w_ug, w_d, h_pool, shifts, out_rows)
    d = dy_slot.shape[1]
    E, two_f, _ = w_ug.shape
    f = two_f // 2
    lib = _native.load()
    _tk = _begin("gemm_bwd_dact")
    rc = lib.hm_grouped_gemm_shifted(
        _native.GEMM_BWD_DACT, dy_slot.data_ptr(), _ptr(w_d), _ptr(seg), E, cap, cap, 0, f, d, dh_ptr, 2 * f,
        None, 0, _ptr(h_pool), 2 * f, None, None, _ptr(shifts[4:6]), max_ctas, _stream())
    _end(_tk)
    _native.check(rc, "hm_grouped_gemm_shifted")
    _count(1)
    _gemm_shifted(_native.GEMM_BWD_DX, dh_ptr, w_ug, seg, E, cap, dh_rows, d, 2 * f, out_rows=out_rows,
                  row_shift=shifts[6:8], max_ctas=max_ctas, name="gemm_bwd_dx_p2p")


def grouped_wgrad_multi_shifted(a_ptrs, b_ptrs, M: int, N: int, seg_multi, out, shift_a=None, shift_b=None,
                                shift_stride: int = 0, max_ctas: int = 0, name: str = "gemm_wgrad_multi") -> None:
    """out[e] += sum_j A_j[seg_j(e) + sa_j]^T . B_j[seg_j(e) + sb_j] (fp32 accumulate), the per-segment
    row offsets sa_j = shift_a[j * shift_stride], sb_j likewise (device int32 tensors or None)."""
    lib = _native.load()
    R = len(a_ptrs)
    if R > 16 or out.dtype != torch.float32:
        raise ValueError("grouped_wgrad_multi_shifted: at most 16 segments, fp32 out")
    E = seg_multi.shape[1] - 1
    nbytes = lib.hm_grouped_wgrad_multi_workspace_bytes(E, R)
    ws = torch.empty((nbytes + 128,), dtype=torch.uint8, device=out.device)
    off = (-ws.data_ptr()) % 128
    ws = ws[off:off + nbytes]
    ap = (ctypes.c_void_p * R)(*a_ptrs)
    bp = (ctypes.c_void_p * R)(*b_ptrs)
    rows = (ctypes.c_int * R)(*([1] * R))
    _tk = _begin(name)
    rc = lib.hm_grouped_wgrad_multi_shifted(1, ap, bp, rows, _ptr(seg_multi), R, E, M, N, _ptr(out), N,
                                            _ptr(shift_a), _ptr(shift_b), shift_stride, _ptr(ws), max_ctas,
                                            _stream())
    _end(_tk)
    _native.check(rc, "hm_grouped_wgrad_multi_shifted")
    _count(2)


def signal_peers(flag_ptrs) -> None:
    """+1 (release, system scope) on each listed device counter after this stream's prior work."""
    n = len(flag_ptrs)
    arr = (ctypes.c_ulonglong * max(n, 1))(*flag_ptrs)
    rc = _native.load().hm_signal_peers(arr, n, _stream())
    _native.check(rc, "hm_signal_peers")
    _count(1 if n else 0)


def wait_flags(flags_ptr: int, stride: int, targets) -> None:
    """Stall the current stream until counters flags[i*stride] >= targets[i]."""
    n = len(targets)
    arr = (ctypes.c_uint * max(n, 1))(*targets)
    rc = _native.load().hm_wait_flags(flags_ptr, stride, arr, n, _stream())
    _native.check(rc, "hm_wait_flags")
    _count(1 if n else 0)
