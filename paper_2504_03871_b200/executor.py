"""Zebra-parallel (ZP) executor: runs a ``TaskGraph`` on real devices and returns a MEASURED
``Timeline`` — the B200 replacement for the reference's timing model
``simulate(graph, orders)`` (``/root/reference/pkg/src/zpsim/simulator.py:33``).

One process per GPU. Ranks ``[0, M)`` are attention ranks, ``[M, M+N)`` expert ranks
(``ZpGroupSpec``, ``core.py:70-79``). Each rank owns three CUDA streams — compute, dispatch,
combine (``PAPER.md:198``) — and two NCCL communicators, one per comm lane, so dispatch and
combine transfers overlap compute and each other. Every task of the graph is issued in ONE
global order (the simulated start order of the graph under ``default_orders``), so each
communicator sees its collectives in the same order on every rank (``comm_order``,
``scheduler.py:110-140``). Cross-lane edges of the DAG become CUDA events.

What each task kind does here:
  ATTN_F(l,j)   combine(l-1) + residual, attention block, router, dispatch permute
  DISP_F(l,j)   expert-count all-gather, then NCCL send/recv of the permuted rows to the
                experts' owners (expert ranks, or attention ranks for Asym-EA offloaded experts)
  EXP_F / OFF_EXP_F   grouped SwiGLU FFN over the received rows (expert-major layout)
  COMB_F(l,j)   expert outputs back to their senders
  DISP_B(l,j)   (l = L: final combine + loss gradient + combine-bwd, the zp-full turnaround)
                send of dY rows
  EXP_B / OFF_EXP_B   grouped FFN backward; expert weight grads accumulate in fp32
  COMB_B(l,j)   dX rows back
  ATTN_B(l,j)   router backward + unpermute-sum, residual, attention backward, combine-bwd(l-1)

Expert placement per layer follows the Asym-EA assignment (``expert_owners``): each expert
rank gives its last o_l local experts to the attention ranks, dealt in (expert rank, local
id) order in blocks of o_l*N/M, which reproduces ``offload_scaling``'s shares exactly
(``taskgraph.py:178-194``).

The tensor work goes through a backend object. ``NativeBackend`` (this file) is the product
path: native sm_100a kernels + torch CUDA streams/events. There is no implicit CPU fallback;
the CPU/gloo tests inject their own backend explicitly.
"""

from __future__ import annotations

import contextlib
import math
import os
import time
import warnings
from dataclasses import dataclass, field
from typing import Optional

import torch
import torch.distributed as dist

from .core import ExpertAssignment
from .scheduler import default_orders
from .simulator import MeasuredTimeline, simulate
from .taskgraph import TaskGraph, TaskKind

K = TaskKind


# ---------------------------------------------------------------------------------------------
# placement


def expert_owners(E: int, M: int, N: int, offload: int, loads=None, capacity=None) -> list:
    """Owner rank of every expert of one layer. Base: expert rank M+i owns experts
    [i*E/N, (i+1)*E/N). With offload o, the last o local experts of each expert rank move to
    the attention ranks, dealt in (expert rank, local id) order, o*N/M per attention rank.

    ``loads`` (expected routed rows per expert, e.g. under a skewed router) switches to a
    load-balanced placement: experts by decreasing load go to the expert rank with room (E/N
    each) whose load after taking it, divided by its capacity weight (``capacity[i]``, default 1:
    the per-rank heterogeneity of BASELINE C5), is smallest (LPT), and the o experts each rank
    offloads are the ones whose loads are closest to the rank's mean (the planner prices an
    offloaded expert at an average share, R4). Every expert rank keeps E/N experts, so the
    offload shares of ``offload_scaling`` (``taskgraph.py:178-194``) hold unchanged."""
    per = E // N
    cap = [1.0] * N if capacity is None else [float(c) for c in capacity]
    if len(cap) != N or min(cap) <= 0:
        raise ValueError(f"need {N} positive expert-rank capacity weights, got {capacity}")
    if loads is None and capacity is not None and len(set(cap)) > 1:
        loads = [1] * E  # uniform router: LPT still spreads experts by capacity (ties -> rank order)
    if loads is None:
        local = [[i * per + q for q in range(per)] for i in range(N)]
    else:
        order = sorted(range(E), key=lambda e: (-loads[e], e))
        local = [[] for _ in range(N)]
        tot = [0] * N
        for e in order:  # largest load first, to the rank it loads least (capacity-weighted LPT)
            i = min((i for i in range(N) if len(local[i]) < per),
                    key=lambda i: ((tot[i] + loads[e]) / cap[i], tot[i], i))
            local[i].append(e)
            tot[i] += loads[e]
        if offload:
            for i in range(N):
                mean = sum(loads[e] for e in local[i]) / per
                moved = sorted(sorted(local[i], key=lambda e: (abs(loads[e] - mean), e))[:offload])
                local[i] = sorted(e for e in local[i] if e not in moved) + moved
    owners = [0] * E
    for i in range(N):
        for e in local[i]:
            owners[e] = M + i
    if offload:
        moved = [local[i][q] for i in range(N) for q in range(per - offload, per)]
        block = offload * N // M
        if block * M != offload * N or block < 1:
            raise ValueError(f"offload {offload} does not split evenly over {M} attention ranks")
        for idx, e in enumerate(moved):
            owners[e] = idx // block
    return owners


@dataclass(frozen=True)
class ZpLayerShape:
    """Tensor shape of one MoE transformer layer as executed."""

    E: int
    k: int
    d: int
    f: int
    tokens_per_mb: int  # tokens per micro-batch per attention rank
    heads: int = 0  # attention heads (0 = d // 128)
    attention: bool = True  # include the attention block (False: identity + residual)
    router_skew: float = 0.0  # Zipf exponent of a per-expert router logit bias (Asym-EA sweep, C5)


# ---------------------------------------------------------------------------------------------
# backends


class NativeBackend:
    """Product backend: sm_100a kernels (``ops``) on three CUDA streams of one device."""

    # communication is stream-ordered (NCCL / device flags), so the executor may defer a
    # task's host-blocking half without changing any communicator's op order on the device
    defer_host_sync = True

    def __init__(self, device, max_ctas: int = 0, comm_priority: bool = False):
        from . import ops  # requires the built extension; fails loudly otherwise

        self.ops = ops
        self.device = torch.device(device)
        self.max_ctas = max_ctas
        # comm_priority: the dispatch / combine lanes' kernels (permute with peer stores, combine
        # backward, flags) get the high stream priority, so the CTA scheduler places them ahead
        # of pending GEMM clusters of the compute lane
        prio = {"compute": 0, "dispatch": -1 if comm_priority else 0, "combine": -1 if comm_priority else 0}
        self.streams = {lane: torch.cuda.Stream(self.device, priority=prio[lane])
                        for lane in ("compute", "dispatch", "combine")}
        self.dtype = torch.bfloat16

    # streams / events
    def on(self, lane: str):
        return torch.cuda.stream(self.streams[lane])

    def mark(self):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev

    def wait(self, ev) -> None:
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)

    def host_wait(self, ev) -> None:
        ev.synchronize()

    def elapsed_ns(self, a, b) -> int:
        return int(round(a.elapsed_time(b) * 1e6))

    def synchronize(self) -> None:
        torch.cuda.synchronize(self.device)

    # tensor ops
    def router(self, u, wg, k, bias=None):
        return self.ops.router_topk(u, wg, k, bias)

    def permute(self, u, r):
        x_perm, _row_src, row_of = self.ops.dispatch_permute(u, r)
        return x_perm, row_of

    def counts(self, r):
        return r.counts

    def combine(self, y_perm, row_of, r):
        return self.ops.combine(y_perm, row_of, r.w)

    def combine_bwd(self, dy, y_perm, row_of, r):
        return self.ops.combine_bwd(dy, y_perm, row_of, r.w)

    def router_bwd(self, dx_perm, row_of, r, dw, x_perm, wg_t, x=None):
        dx, _dl, dwg = self.ops.router_bwd(dx_perm, row_of, r, dw, x_perm, wg_t, want_dwg=True, x=x)
        return dx, dwg

    def transpose(self, w):
        return self.ops.transpose_bf16(w)

    def ffn_fwd(self, x, seg, w_ug, w_d):
        return self.ops.grouped_ffn_fwd(x, seg, w_ug, w_d, self.max_ctas)

    def ffn_bwd_acc(self, dy, x, h, act, seg, w_ug, w_d, gw_ug, gw_d):
        return self.ops.grouped_ffn_bwd_acc(dy, x, h, act, seg, w_ug, w_d, gw_ug, gw_d, self.max_ctas)

    def ffn_bwd_data(self, dy, x, h, act, seg, w_ug, w_d):
        return self.ops.grouped_ffn_bwd_data(dy, x, h, act, seg, w_ug, w_d, self.max_ctas)

    def ffn_wgrad_multi(self, parts, seg_lists, gw_ug, gw_d):
        """parts: per micro-batch (dh, x, dy, act); one grouped GEMM per weight over all of them."""
        seg = self.h2d(seg_lists, torch.int32)
        self.ops.grouped_wgrad_multi([p[0] for p in parts], [p[1] for p in parts], seg, gw_ug,
                                     accumulate=True, max_ctas=self.max_ctas, name="gemm_wgrad_ug")
        self.ops.grouped_wgrad_multi([p[2] for p in parts], [p[3] for p in parts], seg, gw_d,
                                     accumulate=True, max_ctas=self.max_ctas, name="gemm_wgrad_down")

    def tensor(self, shape, dtype=None):
        return torch.empty(shape, dtype=dtype or self.dtype, device=self.device)

    def h2d(self, data, dtype):
        """Small host table -> device on the current stream without a host sync (pinned staging;
        the caching host allocator keeps the staging buffer alive until the copy is done)."""
        return torch.as_tensor(data, dtype=dtype).pin_memory().to(self.device, non_blocking=True)

    def seg_tensor(self, offsets):
        return self.h2d(offsets, torch.int32)

    # peer-memory transport (ZpP2PExecutor)
    def permute_p2p(self, u, r, dest_base, dest_start):
        return self.ops.dispatch_permute_p2p(u, r, dest_base, dest_start, keep_local=True)

    def combine_bwd_p2p(self, dy, y_perm, row_of, r, dest_base, dest_start):
        return self.ops.combine_bwd_p2p(dy, y_perm, row_of, r, dest_base, dest_start)

    def ffn_fwd_rows(self, x, seg, w_ug, w_d, out_rows):
        return self.ops.grouped_ffn_fwd_rows(x, seg, w_ug, w_d, out_rows, self.max_ctas)

    def ffn_bwd_data_rows(self, dy, x, h, act, seg, w_ug, w_d, out_rows):
        return self.ops.grouped_ffn_bwd_data_rows(dy, x, h, act, seg, w_ug, w_d, out_rows, self.max_ctas)

    # device-side receive layout + pool-placed activations (ZpP2PExecutor, device_layout)
    def zp_layout(self, *args):
        self.ops.zp_layout(*args)

    def ffn_fwd_pool(self, x_slot, seg, w_ug, w_d, h_pool, act_pool, shifts, out_rows, cap):
        self.ops.grouped_ffn_fwd_pool(x_slot, seg, w_ug, w_d, h_pool, act_pool, shifts, out_rows, cap,
                                      self.max_ctas)

    def ffn_bwd_data_pool(self, dy_slot, seg, w_ug, w_d, h_pool, dh_ptr, dh_rows, shifts, out_rows, cap):
        self.ops.grouped_ffn_bwd_data_pool(dy_slot, seg, w_ug, w_d, h_pool, dh_ptr, dh_rows, shifts, out_rows,
                                           cap, self.max_ctas)

    def ffn_wgrad_pool(self, ug_ab, down_ab, seg_multi, f_shift, gw_ug, gw_d):
        """Layer weight gradients over all micro-batches: dW_ug += dH^T X (dH pool rows shifted),
        dW_d += dY^T act (act pool rows shifted); f_shift: device view, stride 8 ints."""
        d, f = gw_d.shape[1], gw_d.shape[2]
        self.ops.grouped_wgrad_multi_shifted(ug_ab[0], ug_ab[1], 2 * f, d, seg_multi, gw_ug, shift_a=f_shift,
                                             shift_stride=8, max_ctas=self.max_ctas, name="gemm_wgrad_ug")
        self.ops.grouped_wgrad_multi_shifted(down_ab[0], down_ab[1], d, f, seg_multi, gw_d, shift_b=f_shift,
                                             shift_stride=8, max_ctas=self.max_ctas, name="gemm_wgrad_down")

    def signal(self, flag_ptrs):
        self.ops.signal_peers(flag_ptrs)

    def wait_flags(self, flags_ptr, targets):
        self.ops.wait_flags(flags_ptr, 1, targets)


# ---------------------------------------------------------------------------------------------
# per-rank model state


def rms_norm(x):
    return torch.nn.functional.rms_norm(x, (x.shape[-1],), eps=1e-6)


def attention_block(h, wqkv, wo, heads: int, seq: int = 0):
    """u = h + Attn(RMSNorm(h)): fused QKV projection, causal SDPA, output projection (torch /
    cuBLAS / flash attention; not one of the four hot-path kernels). Pre-norm, as in Mixtral.
    The T rows are one causal sequence, or T / seq independent sequences of `seq` tokens."""
    T, d = h.shape
    hd = d // heads
    S = seq if seq else T
    B = T // S
    qkv = (rms_norm(h) @ wqkv).view(B, S, 3, heads, hd).permute(2, 0, 3, 1, 4)  # [3, B, H, S, hd]
    o = torch.nn.functional.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2], is_causal=True)
    return h + o.permute(0, 2, 1, 3).reshape(T, d) @ wo


@dataclass
class RankState:
    """Parameters (and fp32 gradient accumulators) resident on one rank."""

    owners: list  # per layer: owner rank of each expert
    own: list  # per layer: sorted expert ids owned by this rank
    w_ug: dict = field(default_factory=dict)  # layer -> [E_own, 2f, d]
    w_d: dict = field(default_factory=dict)
    gw_ug: dict = field(default_factory=dict)  # fp32 accumulators
    gw_d: dict = field(default_factory=dict)
    wg: dict = field(default_factory=dict)  # attention ranks: router [d, E]
    bias: dict = field(default_factory=dict)  # attention ranks: router logit bias [E] fp32 or None
    gwg: dict = field(default_factory=dict)
    wqkv: dict = field(default_factory=dict)
    wo: dict = field(default_factory=dict)


class ZpExecutor:
    """Executes one ZP training iteration per ``run()`` on this rank."""

    def __init__(self, graph: TaskGraph, shape: ZpLayerShape, M: int, N: int, rank: int,
                 backend, disp_group=None, comb_group=None, seed: int = 0,
                 durations_hint: Optional[dict] = None, expert_loads=None, expert_capacity=None):
        if graph.mode not in ("zp-full", "distep"):
            raise ValueError("the executor runs zp-full graphs (layer-L experts + loss turnaround) "
                             "or their DistEP lockstep ablation")
        if shape.E % N:
            raise ValueError("N must divide E")
        self.g, self.s, self.M, self.N, self.rank = graph, shape, M, N, rank
        self.W = M + N
        self.be = backend
        self.disp_group, self.comb_group = disp_group, comb_group
        self.is_attn = rank < M
        self.L, self.R = graph.layers, graph.microbatches
        self.heads = shape.heads or max(1, shape.d // 128)
        self.orders = default_orders(graph)
        self.issue_order = self._issue_order()
        owners = [expert_owners(shape.E, M, N, o, expert_loads, expert_capacity) for o in graph.assignment.offload]
        own = [sorted(e for e in range(shape.E) if ow[e] == rank) for ow in owners]
        self.st = RankState(owners=owners, own=own)
        self.wg_t = {}
        self.keep_input_grads = False  # keep dL/d(input) of every micro-batch (input_grads[j])
        self.input_grads = {}
        self._init_params(seed)
        # Initialise both communicators with one collective call by EVERY rank: NCCL requires the
        # first operation on a group to involve all its ranks, and an exchange can involve only
        # some (a layer whose experts all moved to the attention ranks leaves the expert ranks
        # out of that layer's combine) — without this, that first exchange deadlocks.
        for grp in {id(g_): g_ for g_ in (disp_group, comb_group)}.values():
            t = backend.tensor((1,), torch.int32).zero_()
            dist.all_reduce(t, group=grp)

    # ------------------------------------------------------------------ setup
    def _issue_order(self):
        tl = simulate(self.g, self.orders)
        return sorted(self.g.tasks, key=lambda t: (tl.starts[t.id], t.id))

    def _init_params(self, seed: int) -> None:
        s, be, st = self.s, self.be, self.st
        # parameters come from one global seed, generated on the backend's device type, so
        # every rank draws the identical sequence and keeps its own slice
        gen = torch.Generator(device=be.device).manual_seed(seed)

        def rand(shape, std):
            return (torch.randn(shape, generator=gen, device=be.device) * std).to(be.dtype)

        for l in range(1, self.L + 1):
            wqkv = rand((s.d, 3 * s.d), s.d ** -0.5)
            wo = rand((s.d, s.d), s.d ** -0.5)
            wg = rand((s.d, s.E), s.d ** -0.5)
            w_ug_all = rand((s.E, 2 * s.f, s.d), s.d ** -0.5)
            w_d_all = rand((s.E, s.d, s.f), s.f ** -0.5)
            if self.is_attn:
                st.wqkv[l] = wqkv.to(be.device).requires_grad_()
                st.wo[l] = wo.to(be.device).requires_grad_()
                st.wg[l] = wg.to(be.device)
                st.bias[l] = None
                if s.router_skew:
                    from .configs import zipf_bias

                    st.bias[l] = torch.tensor(zipf_bias(s.E, s.router_skew), dtype=torch.float32,
                                              device=be.device)
                st.gwg[l] = torch.zeros((s.d, s.E), dtype=torch.float32, device=be.device)
            own = st.own[l - 1]
            if own:
                idx = torch.tensor(own, device=be.device)
                st.w_ug[l] = w_ug_all[idx].contiguous().to(be.device)
                st.w_d[l] = w_d_all[idx].contiguous().to(be.device)
                st.gw_ug[l] = torch.zeros(st.w_ug[l].shape, dtype=torch.float32, device=be.device)
                st.gw_d[l] = torch.zeros(st.w_d[l].shape, dtype=torch.float32, device=be.device)
        # synthetic inputs / output gradient per micro-batch (attention ranks)
        self.inputs, self.out_grads = {}, {}
        if self.is_attn:
            g2 = torch.Generator(device=be.device).manual_seed(seed * 7919 + 17 + self.rank)
            for j in range(1, self.R + 1):
                self.inputs[j] = torch.randn((s.tokens_per_mb, s.d), generator=g2, device=be.device).to(be.dtype)
                self.out_grads[j] = torch.randn((s.tokens_per_mb, s.d), generator=g2, device=be.device).to(be.dtype)

    # ------------------------------------------------------------------ helpers
    def _ev(self, key):
        return self.events.get(key)

    def _recv_layout(self, l: int, counts_all, rank: Optional[int] = None):
        """Expert-major receive layout on `rank` (default: this rank) for layer l: for each
        owned expert, the rows of every attention rank in rank order. Returns (segment offsets
        per owned expert, {(a, e): (recv_off, rows)})."""
        seg = [0]
        pos = {}
        off = 0
        owners = self.st.owners[l - 1]
        me = self.rank if rank is None else rank
        for e in (e for e in range(self.s.E) if owners[e] == me):
            for a in range(self.M):
                c = counts_all[a][e]
                pos[(a, e)] = (off, c)
                off += c
            seg.append(off)
        return seg, pos

    def _disp_f(self, l, j):
        """DISP_F, first half: enqueue the expert-count all-gather over the dispatch group.
        The second half (`_disp_f_finish`: the host reads the counts — the one host sync per
        (layer, micro-batch), since the receive layout sizes the owners' buffers and GEMM
        launches — then the row transfer) is deferred by the issue loop until a later task
        needs it, so the host keeps issuing other streams' work while the counts travel."""
        s, be = self.s, self.be
        mine = self.my_counts.get((l, j))
        if mine is None:
            mine = be.tensor((s.E,), torch.int32).zero_()
        gathered = [be.tensor((s.E,), torch.int32) for _ in range(self.W)]
        dist.all_gather(gathered, mine.to(torch.int32), group=self.disp_group)
        return lambda: self._disp_f_finish(l, j, gathered)

    def _counts_wait(self, l, j, gathered):
        t0 = time.perf_counter()
        allc = torch.stack(gathered).cpu()
        self.host_wait_s += time.perf_counter() - t0
        counts_all = [[int(v) for v in allc[a].tolist()] for a in range(self.M)]
        self.counts[(l, j)] = counts_all
        return counts_all

    def _send_offsets(self, counts_row):
        off, acc = [], 0
        for c in counts_row:
            off.append(acc)
            acc += c
        return off

    def _exchange(self, l, j, buf_send, buf_recv, forward: bool, group):
        """One all-to-all of rows between attention ranks and owners.

        forward=True: attention rank a sends rows of expert e (its permuted buffer) to
        owner[e]; owners receive expert-major. forward=False: the reverse."""
        owners = self.st.owners[l - 1]
        counts_all = self.counts[(l, j)]
        ops_ = []
        me = self.rank
        for e in range(self.s.E):
            o = owners[e]
            for a in range(self.M):
                c = counts_all[a][e]
                if c == 0:
                    continue
                s_off = self.send_off[(l, j, a)][e]
                if o == me:
                    r_off, _ = self.recv_pos[(l, j)][(a, e)]
                if forward:
                    if a == me and o == me:
                        buf_recv[r_off:r_off + c].copy_(buf_send[s_off:s_off + c])
                    elif a == me:
                        ops_.append(dist.P2POp(dist.isend, buf_send[s_off:s_off + c], o, group=group))
                    elif o == me:
                        ops_.append(dist.P2POp(dist.irecv, buf_recv[r_off:r_off + c], a, group=group))
                else:
                    if a == me and o == me:
                        buf_recv[s_off:s_off + c].copy_(buf_send[r_off:r_off + c])
                    elif o == me:
                        ops_.append(dist.P2POp(dist.isend, buf_send[r_off:r_off + c], a, group=group))
                    elif a == me:
                        ops_.append(dist.P2POp(dist.irecv, buf_recv[s_off:s_off + c], o, group=group))
        if ops_:
            for w in dist.batch_isend_irecv(ops_):
                w.wait()

    # ------------------------------------------------------------------ task handlers
    def _attn_f(self, l, j):
        s, st, be = self.s, self.st, self.be
        if l == 1:
            h = self.inputs[j].detach().requires_grad_()
        else:
            y = be.combine(self.y_perm[(l - 1, j)], self.row_of[(l - 1, j)], self.route[(l - 1, j)])
            h = (self.u[(l - 1, j)].detach() + y).requires_grad_()
        self.h_in[(l, j)] = h
        with torch.enable_grad():
            u = attention_block(h, st.wqkv[l], st.wo[l], self.heads) if s.attention else h * 1
            z = rms_norm(u)  # pre-norm MoE input
        self.u[(l, j)] = u
        self.z[(l, j)] = z
        zd = z.detach()
        r = be.router(zd, st.wg[l], s.k, st.bias[l])
        self.route[(l, j)] = r
        self.my_counts[(l, j)] = be.counts(r)
        self.zd[(l, j)] = zd
        self._attn_permute(l, j, zd, r)

    def _attn_permute(self, l, j, zd, r):
        x_perm, row_of = self.be.permute(zd, r)
        self.row_of[(l, j)], self.x_perm[(l, j)] = row_of, x_perm

    def _disp_f_finish(self, l, j, gathered):
        s, be = self.s, self.be
        counts_all = self._counts_wait(l, j, gathered)
        for a in range(self.M):
            self.send_off[(l, j, a)] = self._send_offsets(counts_all[a])
        seg, pos = self._recv_layout(l, counts_all)
        self.recv_pos[(l, j)] = pos
        self.seg[(l, j)] = seg
        rows = seg[-1]
        self.x_recv[(l, j)] = x_recv = be.tensor((max(rows, 1), s.d))
        self._exchange(l, j, self.x_perm.get((l, j)), x_recv, True, self.disp_group)

    def _exp_f(self, l, j):
        st, be = self.st, self.be
        if not st.own[l - 1]:  # every expert of this rank is offloaded at this layer
            return
        seg = self.seg[(l, j)]
        self.seg_t[(l, j)] = seg_t = be.seg_tensor(seg)
        x = self.x_recv[(l, j)][: max(seg[-1], 1)]
        y, h, act = be.ffn_fwd(x, seg_t, st.w_ug[l], st.w_d[l])
        self.y_recv[(l, j)], self.h_save[(l, j)], self.act[(l, j)] = y, h, act

    def _comb_f(self, l, j):
        s, be = self.s, self.be
        if self.is_attn:
            self.y_perm[(l, j)] = be.tensor((s.tokens_per_mb * s.k, s.d))
        self._exchange(l, j, self.y_recv.get((l, j)), self.y_perm.get((l, j)), False, self.comb_group)

    def _disp_b(self, l, j):
        s, be = self.s, self.be
        if self.is_attn and l == self.L:
            # zp-full loss turnaround on the attention device: final combine, loss gradient,
            # combine backward (the reference prices this attention-side work at 0 ns).
            r = self.route[(l, j)]
            dh = self.out_grads[j]
            self.dh_next[(l, j)] = dh
            dy_perm, dw = be.combine_bwd(dh, self.y_perm[(l, j)], self.row_of[(l, j)], r)
            self.dy_perm[(l, j)], self.dw[(l, j)] = dy_perm, dw
        rows = self.seg[(l, j)][-1]
        self.dy_recv[(l, j)] = dy_recv = be.tensor((max(rows, 1), s.d))
        self._exchange(l, j, self.dy_perm.get((l, j)), dy_recv, True, self.disp_group)

    def _exp_b(self, l, j):
        """Data gradients now; the layer's weight gradients once, after its last micro-batch:
        one grouped GEMM over all R micro-batches (K concatenation) instead of an fp32
        read-modify-write of every expert gradient per micro-batch."""
        st, be = self.st, self.be
        if not st.own[l - 1]:
            return
        seg = self.seg[(l, j)]
        n = max(seg[-1], 1)
        dy = self.dy_recv[(l, j)][:n]
        dx, dh = be.ffn_bwd_data(dy, self.x_recv[(l, j)][:n], self.h_save[(l, j)], self.act[(l, j)],
                                 self.seg_t[(l, j)], st.w_ug[l], st.w_d[l])
        self.dx_recv[(l, j)] = dx
        self.dh[(l, j)] = dh
        if j == self.R:
            parts, segs = [], []
            for jj in range(1, self.R + 1):
                nn = max(self.seg[(l, jj)][-1], 1)
                parts.append((self.dh[(l, jj)], self.x_recv[(l, jj)][:nn], self.dy_recv[(l, jj)][:nn],
                              self.act[(l, jj)]))
                segs.append(self.seg[(l, jj)])
            be.ffn_wgrad_multi(parts, segs, st.gw_ug[l], st.gw_d[l])
            for jj in range(1, self.R + 1):  # the layer's backward activations are done
                self.dh.pop((l, jj), None)
                self.h_save.pop((l, jj), None)

    def _comb_b(self, l, j):
        s, be = self.s, self.be
        if self.is_attn:
            self.dx_perm[(l, j)] = be.tensor((s.tokens_per_mb * s.k, s.d))
        self._exchange(l, j, self.dx_recv.get((l, j)), self.dx_perm.get((l, j)), False, self.comb_group)

    def _attn_b(self, l, j):
        st, be = self.st, self.be
        r = self.route[(l, j)]
        u, z = self.u[(l, j)], self.z[(l, j)]
        key = (st.wg[l]._version, st.wg[l].data_ptr())  # Wg^T kept across iterations until Wg changes
        if self.wg_t.get(l, (None,))[0] != key:
            self.wg_t[l] = (key, be.transpose(st.wg[l]))
        dz, dwg = be.router_bwd(self.dx_perm[(l, j)], self.row_of[(l, j)], r, self.dw[(l, j)],
                                self.x_perm[(l, j)], self.wg_t[l][1], x=self.zd[(l, j)])
        st.gwg[l] += dwg.float()
        h = self.h_in[(l, j)]
        with torch.enable_grad():
            # residual path (dh_next into u) + MoE path (dz through the pre-norm)
            torch.autograd.backward([u, z], [self.dh_next[(l, j)], dz.to(z.dtype)])
        dh = h.grad
        if l > 1:
            self.dh_next[(l - 1, j)] = dh
            self._attn_combine_bwd(l - 1, j, dh)
        elif self.keep_input_grads:  # the iteration's result for a caller that reads it back
            self.input_grads[j] = dh
        # free the layer's activations early
        self.u.pop((l, j), None)
        self.z.pop((l, j), None)
        self.zd.pop((l, j), None)
        self.h_in.pop((l, j), None)

    def _attn_combine_bwd(self, l, j, dh):
        dy_perm, dw = self.be.combine_bwd(dh, self.y_perm[(l, j)], self.row_of[(l, j)], self.route[(l, j)])
        self.dy_perm[(l, j)], self.dw[(l, j)] = dy_perm, dw

    _HANDLERS = {
        K.ATTN_F: ("_attn_f", "compute", "attn"),
        K.DISP_F: ("_disp_f", "dispatch", "all"),
        K.EXP_F: ("_exp_f", "compute", "exp"),
        K.OFF_EXP_F: ("_exp_f", "compute", "attn"),
        K.COMB_F: ("_comb_f", "combine", "all"),
        K.DISP_B: ("_disp_b", "dispatch", "all"),
        K.EXP_B: ("_exp_b", "compute", "exp"),
        K.OFF_EXP_B: ("_exp_b", "compute", "attn"),
        K.COMB_B: ("_comb_b", "combine", "all"),
        K.ATTN_B: ("_attn_b", "compute", "attn"),
    }

    def _participates(self, task) -> bool:
        _, _, who = self._HANDLERS[task.kind]
        if who == "all":
            return True
        if task.kind in (K.OFF_EXP_F, K.OFF_EXP_B):
            return self.is_attn and bool(self.st.own[task.layer - 1])
        return (who == "attn") == self.is_attn

    def _debug_check(self, task) -> None:
        """HM_ZP_DEBUG=1: synchronise after every task and check its outputs are finite."""
        self.be.synchronize()
        key = (task.layer, task.microbatch)
        for name in ("u", "x_perm", "x_recv", "y_recv", "y_perm", "dy_perm", "dy_recv", "dx_recv", "dx_perm"):
            t = getattr(self, name).get(key)
            if t is not None and t.numel() and not bool(torch.isfinite(t.float()).all()):
                raise FloatingPointError(f"rank {self.rank}: non-finite {name} after {task.kind.value} "
                                         f"L{task.layer} M{task.microbatch}")
        r = self.route.get(key)
        if r is not None and (int(r.idx.min()) < 0 or int(r.idx.max()) >= self.s.E):
            raise IndexError(f"rank {self.rank}: router index out of range at L{task.layer} M{task.microbatch}")

    # ------------------------------------------------------------------ iteration
    def _host_preds(self, tasks, preds):
        """Per task, the nearest ancestors this rank takes part in: a task may need host state
        (e.g. the receive layout) from a local task two edges up, through a task it skips."""
        mine = {t.id for t in tasks}
        near: dict = {}

        def nearest(tid):
            stack, acc, seen = list(preds[tid]), set(), set()
            while stack:
                p = stack.pop()
                if p in seen:
                    continue
                seen.add(p)
                if p in mine:
                    acc.add(p)
                else:
                    stack.extend(preds[p])
            return acc

        for t in tasks:
            near[t.id] = nearest(t.id)
        return near

    def _issue(self, task, preds, marks, pending, host_preds) -> None:
        """Issue one task on its lane's stream after its dependencies' events. Deferred halves of
        earlier tasks run first when this task depends on them or shares their lane."""
        be = self.be
        meth, lane, _ = self._HANDLERS[task.kind]
        for pid in [p for p, (_, pl, _) in pending.items() if pl == lane or p in host_preds[task.id]]:
            self._finish(pid, pending, marks)
        with be.on(lane):
            for p in preds[task.id]:
                be.wait(self.events.get(p))
            start = be.mark()
            fin = getattr(self, meth)(task.layer, task.microbatch)
            if fin is not None:
                pending[task.id] = (fin, lane, start)
                if not getattr(be, "defer_host_sync", False):
                    self._finish(task.id, pending, marks)
                return
            end = be.mark()
        self.events[task.id] = end
        marks[task.id] = (start, end)

    def _finish(self, tid, pending, marks) -> None:
        fin, lane, start = pending.pop(tid)
        with self.be.on(lane):
            fin()
            end = self.be.mark()
        self.events[tid] = end
        marks[tid] = (start, end)

    def run(self) -> dict:
        """One forward+backward iteration. Returns {task_id: (start_ns, end_ns)} measured on
        this rank (relative to the iteration start event), for the tasks it took part in."""
        self.events, marks = {}, {}
        for name in ("u", "z", "zd", "h_in", "route", "row_of", "x_perm", "my_counts", "counts", "send_off",
                     "recv_pos", "seg", "seg_t", "x_recv", "y_recv", "h_save", "act", "y_perm",
                     "dy_perm", "dw", "dh_next", "dy_recv", "dx_recv", "dx_perm", "dh"):
            setattr(self, name, {})
        self.host_wait_s = 0.0
        for gdict in (self.st.gw_ug, self.st.gw_d, self.st.gwg):
            for t in gdict.values():
                t.zero_()
        be = self.be
        be.synchronize()
        if dist.is_initialized():
            dist.barrier(group=self.disp_group)  # common time origin (up to launch skew)
        with be.on("compute"):
            t0 = be.mark()
        preds = {t.id: list(self.g.predecessors(t.id)) for t in self.g.tasks}
        debug = os.environ.get("HM_ZP_DEBUG") == "1"
        mine = [t for t in self.issue_order if self._participates(t)]
        host_preds = self._host_preds(mine, preds)
        pending: dict = {}
        for task in mine:
            self._issue(task, preds, marks, pending, host_preds)
            if debug:
                for pid in list(pending):
                    self._finish(pid, pending, marks)
                self._debug_check(task)
        for pid in list(pending):
            self._finish(pid, pending, marks)
        be.synchronize()
        out = {tid: (be.elapsed_ns(t0, a), be.elapsed_ns(t0, b)) for tid, (a, b) in marks.items()}
        return out


# ---------------------------------------------------------------------------------------------
# peer-memory (NVLink) transport


def p2p_dispatch_dest(owners, recv_pos_by_rank, a: int, E: int):
    """Sender side of the fused dispatch for attention rank a: per expert, the owner rank and the
    first row of a's rows inside the owner's expert-major receive buffer."""
    dest_rank = [owners[e] for e in range(E)]
    dest_start = [recv_pos_by_rank[owners[e]][(a, e)][0] for e in range(E)]
    return dest_rank, dest_start


def p2p_return_rows(recv_pos, send_off_by_rank):
    """Owner side of the fused return: for every received row (expert-major order) the attention
    rank it came from and its row in that rank's permuted buffer, so the owner's last GEMM can
    store the row straight back (numpy arrays; rows in receive order)."""
    import numpy as np

    n = sum(c for _, c in recv_pos.values())
    ranks = np.zeros(n, dtype=np.int64)
    rows = np.zeros(n, dtype=np.int64)
    for (a, e), (off, c) in recv_pos.items():
        if c:
            ranks[off:off + c] = a
            rows[off:off + c] = send_off_by_rank[a][e] + np.arange(c)
    return ranks, rows


class PeerArena:
    """Symmetric device memory over all ranks of `group` (torch symmetric memory: the same
    allocation mapped into every peer over NVLink), carved into per-(layer, micro-batch) slots:

      [flags: 4 kinds x W uint32 counters | per (l, j): x | dy (owner receive, `cap` rows each)
                                               | y | dx (attention receive, T*k rows each)]

    Every rank has the same layout, so a slot's offset is rank-independent and a peer's slot
    address is ``ptrs[peer] + offset``. Flag counters are monotonic over the arena's lifetime."""

    FLAG_BYTES = 4096
    DF, CF, DB, CB = range(4)

    def __init__(self, L: int, R: int, cap: int, tk: int, d: int, W: int, group, device):
        import torch.distributed._symmetric_memory as symm

        self.L, self.R, self.cap, self.tk, self.d, self.W = L, R, cap, tk, d, W
        self.rb = d * 2
        self.slot_bytes = (2 * cap + 2 * tk) * self.rb
        nbytes = self.FLAG_BYTES + L * R * self.slot_bytes
        self.buf = symm.empty(nbytes, dtype=torch.uint8, device=device)
        self.handle = symm.rendezvous(self.buf, group)
        self.ptrs = [int(p) for p in self.handle.buffer_ptrs]
        self.rank = self.handle.rank
        self.buf[: self.FLAG_BYTES].zero_()
        torch.cuda.synchronize(device)
        dist.barrier(group=group)

    @classmethod
    def bytes_needed(cls, L: int, R: int, cap: int, tk: int, d: int) -> int:
        return cls.FLAG_BYTES + L * R * (2 * cap + 2 * tk) * d * 2

    def offset(self, l: int, j: int, which: str) -> int:
        base = self.FLAG_BYTES + ((l - 1) * self.R + (j - 1)) * self.slot_bytes
        cap, tk, rb = self.cap, self.tk, self.rb
        return base + {"x": 0, "dy": cap * rb, "y": 2 * cap * rb, "dx": (2 * cap + tk) * rb}[which]

    def view(self, l, j, which, rows):
        off = self.offset(l, j, which)
        return self.buf[off:off + rows * self.rb].view(torch.bfloat16).view(rows, self.d)

    def addr(self, rank, l, j, which) -> int:
        return self.ptrs[rank] + self.offset(l, j, which)

    def flag_addr(self, rank, kind, sender) -> int:
        return self.ptrs[rank] + (kind * self.W + sender) * 4

    def local_flags(self, kind) -> int:
        return self.ptrs[self.rank] + kind * self.W * 4


class ZpP2PExecutor(ZpExecutor):
    """ZP executor whose dispatch / combine move rows over NVLink peer memory instead of NCCL
    send/recv, each fused into the kernel that produces the rows:

      DISP_F  permute kernel stores every routed row straight into its owner's receive slot
      EXP_F   the down-projection GEMM epilogue stores each output row into its sender's y slot
      DISP_B  combine-backward kernel stores w*dY rows into the owners' dy slots
      EXP_B   the dX GEMM epilogue stores each row into its sender's dx slot

    A transfer completes with a release add on the receiver's flag counter (one per kind and
    sender) after the producing kernel; the receiver's stream waits (acquire) for the count of
    exchanges it expects. Only the expert-count all-gather (one per layer and micro-batch, as in
    the NCCL path) stays a collective. Same task graph, streams and issue order as ZpExecutor.

    device_layout (default; HM_ZP_HOST_LAYOUT=1 restores the host path): the all-gathered counts
    never reach the host. One ``hm_zp_layout`` kernel per (layer, micro-batch), on the dispatch
    stream right after the count all-gather, computes every sender's destination rows, the
    owner's expert segments and per-row return addresses, and bump-allocates the micro-batch's
    saved activations (h, act; dH shares their row numbering) in a per-layer region of a pool
    sized HM_ZP_POOL_FACTOR (1.25) x the expected rows (capped at the worst case and by free memory).
    The expert GEMMs read the segment table and pool row shifts from device memory and are sized
    by the receive capacity; a pool overflow is flagged on the device and raised after the step."""

    def __init__(self, graph, shape, M, N, rank, backend, disp_group=None, comb_group=None,
                 seed: int = 0, durations_hint=None, expert_loads=None, expert_capacity=None,
                 device_layout: Optional[bool] = None):
        super().__init__(graph, shape, M, N, rank, backend, disp_group, comb_group, seed, durations_hint,
                         expert_loads, expert_capacity)
        self.expert_loads = expert_loads
        if self.W > 8:
            raise ValueError("p2p transport supports at most 8 ranks (one NVSwitch domain)")
        s = shape
        max_own = max(sum(1 for o in ow if o == r) for ow in self.st.owners for r in range(self.W))
        cap = s.tokens_per_mb * M * min(s.k, max_own)  # worst case rows one owner can receive
        self.arena = PeerArena(self.L, self.R, cap, s.tokens_per_mb * s.k, s.d, self.W,
                               disp_group, backend.device)
        if self.arena.rank != rank:
            raise ValueError("the dispatch group must rank processes like the world")
        self.expected = [[0] * self.W for _ in range(4)]  # per kind, per sender: exchanges seen
        self.owner_sets = [sorted(set(ow)) for ow in self.st.owners]
        if device_layout is None:
            device_layout = os.environ.get("HM_ZP_HOST_LAYOUT") != "1" and hasattr(backend, "zp_layout")
        self.device_layout = bool(device_layout)
        if self.device_layout:
            self._init_device_layout()

    def _alloc_pools(self) -> None:
        """Per-layer pool regions for the saved expert activations of its R micro-batches:
        pool_factor x the expected rows (the router's per-expert loads when known, else uniform
        routing), capped at the worst case; dH shares the row numbering, one layer at a time."""
        s, be, st = self.s, self.be, self.st
        M, R, E = self.M, self.R, s.E
        loads = self.expert_loads
        share = [1.0 / E] * E if not loads or sum(loads) <= 0 else [v / sum(loads) for v in loads]

        def regions(factor):
            bases, rows_l, base = [], [], 0
            for own in st.own:
                rows = 0
                if own:
                    worst = R * s.tokens_per_mb * M * min(s.k, len(own))
                    expect = R * s.tokens_per_mb * M * s.k * sum(share[e] for e in own)
                    rows = min(worst, int(math.ceil(factor * expect / 128.0)) * 128)
                bases.append(base)
                rows_l.append(rows)
                base += rows
            return bases, rows_l, base

        self.h_pool = self.act_pool = self.dh_pool = None  # release before reallocating
        bases, rows_l, base = regions(self.pool_factor)
        row_bytes = 3 * s.f * 2  # h + act per pool row; dH: one layer's rows
        need = base * row_bytes + max(rows_l) * 2 * s.f * 2
        if be.device.type == "cuda":
            # fit the pools in what the device has left (8 GiB headroom for the step's transients)
            torch.cuda.empty_cache()
            free = torch.cuda.mem_get_info(be.device)[0] - (8 << 30)
            if need > free:
                fit = self.pool_factor * free / need
                if fit < 1.0:
                    raise RuntimeError(f"rank {self.rank}: activation pools need {need / 2**30:.1f} GiB at the "
                                       f"expected routed rows, {free / 2**30:.1f} GiB free")
                warnings.warn(f"rank {self.rank}: pool factor {self.pool_factor:.2f} -> {fit:.2f} to fit memory")
                self.pool_factor = fit
                bases, rows_l, base = regions(fit)
        self.pool_base, self.pool_rows = bases, rows_l
        self.h_pool = be.tensor((max(base, 1), 2 * s.f))
        self.act_pool = be.tensor((max(base, 1), s.f))
        self.dh_pool = be.tensor((max(max(self.pool_rows), 1), 2 * s.f))

    def _init_device_layout(self) -> None:
        s, be, ar, st = self.s, self.be, self.arena, self.st
        L, R, M, W, E = self.L, self.R, self.M, self.W, s.E
        dev = be.device
        self.n_own = [len(o) for o in st.own]
        self.pool_factor = float(os.environ.get("HM_ZP_POOL_FACTOR", "1.25"))
        self._alloc_pools()
        i32, i64 = torch.int32, torch.int64
        self.owners_t = torch.tensor(st.owners, dtype=i32, device=dev)
        lj = [(l, j) for l in range(1, L + 1) for j in range(1, R + 1)]
        self.y_base_t = torch.tensor([[ar.addr(a, l, j, "y") for a in range(M)] for l, j in lj],
                                     dtype=i64, device=dev).view(L, R, M)
        self.dx_delta = ar.offset(1, 1, "dx") - ar.offset(1, 1, "y")
        self.dest_x_t = torch.tensor([[ar.addr(st.owners[l - 1][e], l, j, "x") for e in range(E)] for l, j in lj],
                                     dtype=i64, device=dev).view(L, R, E)
        self.dest_dy_t = torch.tensor([[ar.addr(st.owners[l - 1][e], l, j, "dy") for e in range(E)] for l, j in lj],
                                      dtype=i64, device=dev).view(L, R, E)
        self.dest_start_t = torch.zeros((L, R, E), dtype=i32, device=dev)
        self.seg_l = [torch.zeros((R, n + 1), dtype=i32, device=dev) if n else None for n in self.n_own]
        self.out_rows_y_t = torch.zeros((L, R, ar.cap), dtype=i64, device=dev)
        self.out_rows_dx_t = torch.zeros((L, R, ar.cap), dtype=i64, device=dev)
        self.shifts_t = torch.zeros((L, R, 8), dtype=i32, device=dev)
        self.top_t = torch.zeros((L,), dtype=i32, device=dev)
        self.err_t = torch.zeros((1,), dtype=i32, device=dev)
        self.counts_t = torch.zeros((L, R, W, E), dtype=i32, device=dev)

    # signalling helpers
    def _signal(self, kind, receivers):
        a = self.arena
        self.be.signal([a.flag_addr(r, kind, self.rank) for r in receivers])

    def _wait(self, kind, senders):
        exp = self.expected[kind]
        for s_ in senders:
            exp[s_] += 1
        self.be.wait_flags(self.arena.local_flags(kind), exp)

    # task handlers
    def _attn_permute(self, l, j, zd, r):
        pass  # the permute runs fused with the dispatch, once the receive layout is known

    def _disp_f(self, l, j):
        if not self.device_layout:
            return super()._disp_f(l, j)
        # count all-gather, then the receive layout on the device: no host read of the counts
        s, be, ar = self.s, self.be, self.arena
        mine = self.my_counts.get((l, j))
        if mine is None:
            mine = be.tensor((s.E,), torch.int32).zero_()
        cnt = self.counts_t[l - 1, j - 1]
        dist.all_gather_into_tensor(cnt, mine.to(torch.int32).contiguous(), group=self.disp_group)
        n = self.n_own[l - 1]
        be.zp_layout(cnt, self.M, self.owners_t[l - 1], self.rank, n, ar.cap, self.y_base_t[l - 1, j - 1],
                     self.dx_delta, ar.rb, self.dest_start_t[l - 1, j - 1],
                     self.seg_l[l - 1][j - 1] if n else None, self.out_rows_y_t[l - 1, j - 1],
                     self.out_rows_dx_t[l - 1, j - 1], self.shifts_t[l - 1, j - 1], self.top_t[l - 1:l],
                     self.pool_base[l - 1], self.pool_rows[l - 1], self.err_t)
        if self.is_attn:
            x_perm, row_of = be.permute_p2p(self.zd[(l, j)], self.route[(l, j)], self.dest_x_t[l - 1, j - 1],
                                            self.dest_start_t[l - 1, j - 1])
            self.x_perm[(l, j)], self.row_of[(l, j)] = x_perm, row_of
            self._signal(ar.DF, self.owner_sets[l - 1])
        if self.st.own[l - 1]:
            self._wait(ar.DF, range(self.M))
        return None

    def _disp_f_finish(self, l, j, gathered):
        s, be, ar = self.s, self.be, self.arena
        counts_all = self._counts_wait(l, j, gathered)
        owners = self.st.owners[l - 1]
        send_off = {a: self._send_offsets(counts_all[a]) for a in range(self.M)}
        pos_by = {o: self._recv_layout(l, counts_all, o)[1] for o in self.owner_sets[l - 1]}
        seg, pos = self._recv_layout(l, counts_all)
        self.seg[(l, j)], self.recv_pos[(l, j)] = seg, pos
        for o, pos_o in pos_by.items():  # the peer stores must stay inside each owner's slot
            need = sum(c for _, c in pos_o.values())
            if need > ar.cap:
                raise RuntimeError(f"layer {l} micro-batch {j}: owner rank {o} would receive {need} rows, "
                                   f"more than its receive slot holds ({ar.cap})")
        if self.is_attn:
            dest_rank, dest_start = p2p_dispatch_dest(owners, pos_by, self.rank, s.E)
            self.dest_start[(l, j)] = st_t = be.h2d(dest_start, torch.int32)
            self.dest_x[(l, j)] = bx = be.h2d([ar.addr(o, l, j, "x") for o in dest_rank], torch.int64)
            self.dest_dy[(l, j)] = be.h2d([ar.addr(o, l, j, "dy") for o in dest_rank], torch.int64)
            x_perm, row_of = be.permute_p2p(self.zd[(l, j)], self.route[(l, j)], bx, st_t)
            self.x_perm[(l, j)], self.row_of[(l, j)] = x_perm, row_of
            self._signal(ar.DF, self.owner_sets[l - 1])
        if seg[-1] or self.st.own[l - 1]:
            if self.st.own[l - 1]:
                self._wait(ar.DF, range(self.M))
            ranks, rows = p2p_return_rows(pos, send_off)
            y_addr = [ar.addr(a, l, j, "y") for a in range(self.M)]
            import numpy as np

            out = np.asarray(y_addr, dtype=np.int64)[ranks] + rows * ar.rb if len(ranks) else np.zeros(1, np.int64)
            self.out_rows[(l, j)] = be.h2d(out, torch.int64)
        self.x_recv[(l, j)] = ar.view(l, j, "x", max(seg[-1], 1))

    def _exp_f(self, l, j):
        st, be = self.st, self.be
        if not st.own[l - 1]:  # every expert of this rank is offloaded at this layer
            return
        if self.device_layout:
            ar = self.arena
            be.ffn_fwd_pool(ar.view(l, j, "x", ar.cap), self.seg_l[l - 1][j - 1], st.w_ug[l], st.w_d[l],
                            self.h_pool, self.act_pool, self.shifts_t[l - 1, j - 1],
                            self.out_rows_y_t[l - 1, j - 1], ar.cap)
            return
        seg = self.seg[(l, j)]
        self.seg_t[(l, j)] = seg_t = be.seg_tensor(seg)
        x = self.x_recv[(l, j)]
        h, act = be.ffn_fwd_rows(x, seg_t, st.w_ug[l], st.w_d[l], self.out_rows[(l, j)])
        self.h_save[(l, j)], self.act[(l, j)] = h, act

    def _comb_f(self, l, j):
        ar = self.arena
        if self.st.own[l - 1]:
            self._signal(ar.CF, range(self.M))
        if self.is_attn:
            self._wait(ar.CF, self.owner_sets[l - 1])
            self.y_perm[(l, j)] = ar.view(l, j, "y", self.s.tokens_per_mb * self.s.k)

    def _attn_combine_bwd(self, l, j, dh):
        pass  # fused with the dY dispatch in DISP_B(l, j)

    def _disp_b(self, l, j):
        be, ar = self.be, self.arena
        if self.is_attn:
            if l == self.L:
                self.dh_next[(l, j)] = self.out_grads[j]
            r = self.route[(l, j)]
            if self.device_layout:
                dest_dy, dest_start = self.dest_dy_t[l - 1, j - 1], self.dest_start_t[l - 1, j - 1]
            else:
                dest_dy, dest_start = self.dest_dy[(l, j)], self.dest_start[(l, j)]
            self.dw[(l, j)] = be.combine_bwd_p2p(self.dh_next[(l, j)], self.y_perm[(l, j)], self.row_of[(l, j)],
                                                 r, dest_dy, dest_start)
            self._signal(ar.DB, self.owner_sets[l - 1])
        if self.st.own[l - 1]:
            self._wait(ar.DB, range(self.M))
        if not self.device_layout:
            self.dy_recv[(l, j)] = ar.view(l, j, "dy", max(self.seg[(l, j)][-1], 1))

    def _exp_b(self, l, j):
        st, be, ar = self.st, self.be, self.arena
        if not st.own[l - 1]:
            return
        if self.device_layout:
            self._exp_b_pool(l, j)
            return
        seg = self.seg[(l, j)]
        if (l, j) not in self.out_rows_dx:
            delta = ar.offset(l, j, "dx") - ar.offset(l, j, "y")
            self.out_rows_dx[(l, j)] = self.out_rows[(l, j)] + delta
        dh = be.ffn_bwd_data_rows(self.dy_recv[(l, j)], self.x_recv[(l, j)], self.h_save[(l, j)],
                                  self.act[(l, j)], self.seg_t[(l, j)], st.w_ug[l], st.w_d[l],
                                  self.out_rows_dx[(l, j)])
        self.dh[(l, j)] = dh
        if j == self.R:
            parts, segs = [], []
            for jj in range(1, self.R + 1):
                parts.append((self.dh[(l, jj)], self.x_recv[(l, jj)], self.dy_recv[(l, jj)], self.act[(l, jj)]))
                segs.append(self.seg[(l, jj)])
            be.ffn_wgrad_multi(parts, segs, st.gw_ug[l], st.gw_d[l])
            for jj in range(1, self.R + 1):
                self.dh.pop((l, jj), None)
                self.h_save.pop((l, jj), None)

    def _exp_b_pool(self, l, j):
        """EXP_B with the device layout: dH lands in the layer's dh buffer addressed by the pool
        rows of this micro-batch (the buffer pointer is moved back by the layer's first pool row),
        dX goes straight back to the senders; after the layer's last micro-batch one grouped GEMM
        per weight forms the layer's weight gradients over all R micro-batches."""
        st, be, ar, s = self.st, self.be, self.arena, self.s
        rb_dh = 2 * s.f * 2
        dh_ptr = self.dh_pool.data_ptr() - self.pool_base[l - 1] * rb_dh
        dh_rows = self.pool_base[l - 1] + self.pool_rows[l - 1]
        be.ffn_bwd_data_pool(ar.view(l, j, "dy", ar.cap), self.seg_l[l - 1][j - 1], st.w_ug[l], st.w_d[l],
                             self.h_pool, dh_ptr, dh_rows, self.shifts_t[l - 1, j - 1],
                             self.out_rows_dx_t[l - 1, j - 1], ar.cap)
        if j == self.R:
            R, me = self.R, self.rank
            ug = ([dh_ptr] * R, [ar.addr(me, l, jj, "x") for jj in range(1, R + 1)])
            down = ([ar.addr(me, l, jj, "dy") for jj in range(1, R + 1)], [self.act_pool.data_ptr()] * R)
            be.ffn_wgrad_pool(ug, down, self.seg_l[l - 1], self.shifts_t[l - 1, :, 1], st.gw_ug[l], st.gw_d[l])

    def _comb_b(self, l, j):
        ar = self.arena
        if self.st.own[l - 1]:
            self._signal(ar.CB, range(self.M))
        if self.is_attn:
            self._wait(ar.CB, self.owner_sets[l - 1])
            self.dx_perm[(l, j)] = ar.view(l, j, "dx", self.s.tokens_per_mb * self.s.k)

    def run(self) -> dict:
        for name in ("dest_start", "dest_x", "dest_dy", "out_rows", "out_rows_dx"):
            setattr(self, name, {})
        if not self.device_layout:
            return super().run()
        for attempt in range(4):
            self.top_t.zero_()
            self.err_t.zero_()
            out = super().run()
            # every rank learns whether any owner's pool overflowed (then a micro-batch was
            # skipped there): grow the pools and run the iteration again
            err = self.err_t.clone()
            dist.all_reduce(err, op=dist.ReduceOp.MAX, group=self.disp_group)
            err = int(err.item())
            if not err:
                return out
            if err & ~1 or attempt == 3:
                raise RuntimeError(f"rank {self.rank}: device receive layout error (code {err}: 1 = activation "
                                   f"pool overflow, 4 = receive slot overflow, 8 = owner outside the exchange) "
                                   f"at HM_ZP_POOL_FACTOR {self.pool_factor}")
            self.pool_factor *= 1.5
            self.pool_regrows = getattr(self, "pool_regrows", 0) + 1
            warnings.warn(f"rank {self.rank}: activation pool overflow; pool factor -> {self.pool_factor:.2f}, "
                          "iteration repeated")
            self._alloc_pools()
        return out


def merge_rank_intervals(graph: TaskGraph, per_rank: list, M: int) -> MeasuredTimeline:
    """Timeline of the representative devices (the reference's one-device-per-role model,
    ``taskgraph.py:6-7``). Each role is represented by ONE rank — its critical rank, the one whose
    last task ends latest — so every lane of the Timeline holds one real stream's intervals and
    never overlaps itself (an envelope over several ranks' intervals would, and would push
    ``compute_metrics``' utilisation above 1 for M > 1). A task the representative did not take
    part in takes its interval from the role's other ranks, or from any rank that ran it (e.g. a
    communication task whose home role had nothing to send). The makespan is the latest end on
    any rank."""
    W = len(per_rank)
    roles = {"attn": list(range(0, M)), "exp": list(range(M, W))}

    def last_end(r):
        return max((b for _, b in per_rank[r].values()), default=-1)

    rep = {role: max(rs, key=lambda r: (last_end(r), -r)) for role, rs in roles.items() if rs}
    starts, ends = {}, {}
    for t in graph.tasks:
        home = roles[t.device]
        cands = ([rep[t.device]] if t.device in rep else []) + [r for r in home if r != rep.get(t.device)]
        cands += [r for r in range(W) if r not in home]
        r = next((r for r in cands if t.id in per_rank[r]), None)
        if r is None:
            raise KeyError(f"task {t.id} ({t.kind.value}) ran on no rank")
        starts[t.id], ends[t.id] = per_rank[r][t.id]
    orders = default_orders(graph)
    makespan = max((b for iv in per_rank for _, b in iv.values()), default=0)
    return MeasuredTimeline(starts, ends, makespan, {k: list(v) for k, v in orders.items()},
                            per_rank=list(per_rank), representative_ranks=rep)


def execute(graph: TaskGraph, executor: ZpExecutor, world_group=None) -> MeasuredTimeline:
    """Run one iteration on every rank and return the measured Timeline (all ranks)."""
    local = executor.run()
    W = executor.W
    gathered = [None] * W
    dist.all_gather_object(gathered, local, group=world_group)
    return merge_rank_intervals(graph, gathered, executor.M)
