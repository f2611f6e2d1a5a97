"""CPU (fp32, torch) backend for exercising the ZP executor's host logic and collective
choreography over gloo — TEST INFRASTRUCTURE ONLY (the product backend is
``executor.NativeBackend``; the executor never falls back to this)."""

import contextlib
import time
from dataclasses import dataclass

import torch


@dataclass
class CpuRouting:
    idx: torch.Tensor
    w: torch.Tensor
    counts: torch.Tensor
    offsets: torch.Tensor


class CpuBackend:
    dtype = torch.float32
    device = torch.device("cpu")
    max_ctas = 0

    def on(self, lane):
        return contextlib.nullcontext()

    def mark(self):
        return time.perf_counter_ns()

    def wait(self, ev):
        pass

    def host_wait(self, ev):
        pass

    def elapsed_ns(self, a, b):
        return int(b - a)

    def synchronize(self):
        pass

    def tensor(self, shape, dtype=None):
        return torch.zeros(shape, dtype=dtype or self.dtype)

    def seg_tensor(self, offsets):
        return torch.tensor(offsets, dtype=torch.int32)

    def transpose(self, w):
        return w.t().contiguous()

    # -- routing
    def router(self, u, wg, k, bias=None):
        logits = u.float() @ wg.float()
        if bias is not None:
            logits = logits + bias
        E = wg.shape[1]
        # ties -> lower id: stable descending sort on (-logit, e)
        order = torch.argsort(-logits, dim=1, stable=True)
        idx = order[:, :k]
        w = torch.softmax(torch.gather(logits, 1, idx), dim=1)
        counts = torch.bincount(idx.reshape(-1), minlength=E).to(torch.int32)
        offsets = torch.zeros(E + 1, dtype=torch.int32)
        offsets[1:] = torch.cumsum(counts, 0)
        return CpuRouting(idx.to(torch.int32), w, counts, offsets)

    def counts(self, r):
        return r.counts

    def permute(self, u, r):
        T, k = r.idx.shape
        flat_e = r.idx.reshape(-1).long()
        flat_t = torch.arange(T).repeat_interleave(k)
        key = flat_e * (T + 1) + flat_t
        order = torch.argsort(key, stable=True)
        row_of = torch.empty(T * k, dtype=torch.long)
        row_of[order] = torch.arange(T * k)
        return u[flat_t[order]].contiguous(), row_of.reshape(T, k)

    def combine(self, y_perm, row_of, r):
        T, k = row_of.shape
        return (y_perm[row_of.reshape(-1)].reshape(T, k, -1) * r.w[:, :, None]).sum(1)

    def combine_bwd(self, dy, y_perm, row_of, r):
        T, k = row_of.shape
        dy_perm = torch.zeros_like(y_perm)
        dy_perm[row_of.reshape(-1)] = (r.w[:, :, None] * dy[:, None, :]).reshape(T * k, -1)
        dw = (y_perm[row_of.reshape(-1)].reshape(T, k, -1) * dy[:, None, :]).sum(-1)
        return dy_perm, dw

    def router_bwd(self, dx_perm, row_of, r, dw, x_perm, wg_t, x=None):
        T, k = row_of.shape
        dx = dx_perm[row_of.reshape(-1)].reshape(T, k, -1).sum(1)
        dl = r.w * (dw - (r.w * dw).sum(1, keepdim=True))
        dx = dx + (dl[:, :, None] * wg_t[r.idx.long()]).sum(1)
        E = wg_t.shape[0]
        # each permuted row is a routed copy of one token: dWg[:, e] = sum_rows dl * x_perm
        dl_perm = torch.zeros(T * k)
        dl_perm[row_of.reshape(-1)] = dl.reshape(-1)
        dwg = torch.zeros(x_perm.shape[1], E)
        off = r.offsets.tolist()
        for e in range(E):
            dwg[:, e] = x_perm[off[e]:off[e + 1]].float().t() @ dl_perm[off[e]:off[e + 1]]
        return dx, dwg

    # -- experts (gate/up interleaved in 128-row blocks, as on the GPU)
    @staticmethod
    def _split(w_ug):
        E, two_f, d = w_ug.shape
        f = two_f // 2
        v = w_ug.reshape(E, f // 128, 2, 128, d)
        return v[:, :, 0].reshape(E, f, d), v[:, :, 1].reshape(E, f, d)

    def ffn_fwd(self, x, seg, w_ug, w_d):
        wg, wu = self._split(w_ug)
        seg = seg.tolist()
        ys, hs, acts = [], [], []
        for e in range(len(seg) - 1):
            xe = x[seg[e]:seg[e + 1]]
            g, u = xe @ wg[e].t(), xe @ wu[e].t()
            a = torch.nn.functional.silu(g) * u
            ys.append(a @ w_d[e].t())
            hs.append(torch.cat([g, u], 1))
            acts.append(a)
        cat = lambda xs, n: torch.cat(xs, 0) if xs else torch.zeros(0, n)  # noqa: E731
        f = w_d.shape[2]
        y = cat(ys, w_d.shape[1])
        if y.shape[0] < x.shape[0]:
            y = torch.cat([y, torch.zeros(x.shape[0] - y.shape[0], y.shape[1])])
        return y, cat(hs, 2 * f), cat(acts, f)

    def ffn_bwd_data(self, dy, x, h, act, seg, w_ug, w_d):
        wg, wu = self._split(w_ug)
        seg = seg.tolist()
        f = w_d.shape[2]
        dx = torch.zeros_like(x)
        dh = torch.zeros(x.shape[0], 2 * f)
        for e in range(len(seg) - 1):
            a0, a1 = seg[e], seg[e + 1]
            g, u = h[a0:a1, :f], h[a0:a1, f:]
            da = dy[a0:a1] @ w_d[e]
            sg = torch.sigmoid(g)
            dg = da * u * sg * (1 + g * (1 - sg))
            du = da * torch.nn.functional.silu(g)
            dx[a0:a1] = dg @ wg[e] + du @ wu[e]
            dh[a0:a1] = torch.cat([dg, du], 1)
        return dx, dh

    def ffn_wgrad_multi(self, parts, seg_lists, gw_ug, gw_d):
        f = gw_d.shape[2]
        E = gw_d.shape[0]
        for (dh, x, dy, act), seg in zip(parts, seg_lists):
            for e in range(E):
                a0, a1 = seg[e], seg[e + 1]
                dg, du = dh[a0:a1, :f], dh[a0:a1, f:]
                g_gate = dg.t() @ x[a0:a1]
                g_up = du.t() @ x[a0:a1]
                inter = torch.stack([g_gate.reshape(f // 128, 128, -1), g_up.reshape(f // 128, 128, -1)], 1)
                gw_ug[e] += inter.reshape(2 * f, -1)
                gw_d[e] += dy[a0:a1].t() @ act[a0:a1]

    def ffn_bwd_acc(self, dy, x, h, act, seg, w_ug, w_d, gw_ug, gw_d):
        wg, wu = self._split(w_ug)
        seg = seg.tolist()
        f = w_d.shape[2]
        dx = torch.zeros_like(x)
        dgs, dus = [], []
        for e in range(len(seg) - 1):
            a0, a1 = seg[e], seg[e + 1]
            xe = x[a0:a1].clone().requires_grad_()
            wge = wg[e].clone().requires_grad_()
            wue = wu[e].clone().requires_grad_()
            wde = w_d[e].clone().requires_grad_()
            ye = (torch.nn.functional.silu(xe @ wge.t()) * (xe @ wue.t())) @ wde.t()
            ye.backward(dy[a0:a1])
            dx[a0:a1] = xe.grad
            gw_d[e] += wde.grad
            dgs.append(wge.grad)
            dus.append(wue.grad)
        if dgs:
            E = len(dgs)
            g = torch.stack(dgs).reshape(E, f // 128, 128, -1)
            u = torch.stack(dus).reshape(E, f // 128, 128, -1)
            gw_ug += torch.stack([g, u], 2).reshape(E, 2 * f, -1)
        return dx
