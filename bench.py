"""Benchmark: MoE expert layer forward+backward tokens/s on B200 (BASELINE.json metric).

Workload at N=1: configs[1] = Mixtral-style layer C2 (E=8, top-2, d=4096, f=14336, bf16) with
T=16384 tokens per step, synthetic seeded inputs, random-init weights. One step = router ->
dispatch permute -> grouped SwiGLU FFN -> combine, forward and backward (all weight grads).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2|C3|C1] [--impl reference]

For N > 1 launch with torchrun (one rank per GPU, NCCL); see --mode.
Prints ONE JSON line (rank 0). Timing: CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks; inputs are larger than L2 (no flush needed).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

if int(os.environ.get("WORLD_SIZE", "1")) > 1:
    # NCCL's communicator lines (INFO) go to stderr: main() points fd 1 at stderr and writes
    # the one JSON line to a duplicate of the original stdout
    os.environ.setdefault("NCCL_DEBUG", "INFO")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

METRIC = "MoE layer fwd+bwd tokens/sec"
UNIT = "tokens/s"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(FALLBACK_PEAKS)
    d["source"] = "fallback (B200_PROFILING.md)"
    return d


# ---------------------------------------------------------------------------------------------
# clocks sampler (pynvml) during the timed region


class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int, period: float = 0.02):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.power_w = []
        self.power_source = None
        self.limit_w = None
        self._stop = threading.Event()
        self._thread = None
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            try:
                self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self._h) / 1000.0
            except Exception:  # noqa: BLE001
                self.limit_w = None
        except Exception:  # noqa: BLE001 - clocks are best effort
            self._nv = None

    def _power_w(self):
        # instantaneous board power (NVML_FI_DEV_POWER_INSTANT); nvmlDeviceGetPowerUsage is a
        # ~1 s running average on B200 and lags a sub-second timed region toward idle
        nv = self._nv
        fi = getattr(nv, "NVML_FI_DEV_POWER_INSTANT", None)
        if fi is not None and self.power_source != "average":
            try:
                v = nv.nvmlDeviceGetFieldValues(self._h, [fi])[0]
                if v.nvmlReturn == 0:
                    self.power_source = "instant"
                    return float(v.value.uiVal) / 1000.0
            except Exception:  # noqa: BLE001
                pass
        self.power_source = "average"
        return nv.nvmlDeviceGetPowerUsage(self._h) / 1000.0

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                try:
                    self.power_w.append(self._power_w())
                except Exception:  # noqa: BLE001
                    pass
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        pw = sorted(self.power_w)
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s), "power_w_median": pw[len(pw) // 2] if pw else None,
                "power_limit_w": self.limit_w, "power_source": self.power_source}


# ---------------------------------------------------------------------------------------------


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 and not dist.is_initialized():
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return ws, rank, local


def max_over_ranks(v: float, ws: int) -> float:
    if ws == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws: int):
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()


def make_layer_tensors(cfg, seed: int, device):
    """Random-init bf16 parameters and inputs generated on the device (seeded)."""
    g = torch.Generator(device=device).manual_seed(seed)

    def n(shape, std):
        return (torch.randn(shape, generator=g, device=device, dtype=torch.float32) * std).to(torch.bfloat16)

    E, d, f, T = cfg.E, cfg.d, cfg.f, cfg.T
    x = n((T, d), 1.0)
    wg = n((d, E), d ** -0.5)
    w_ug = n((E, 2 * f, d), d ** -0.5)
    w_down = n((E, d, f), f ** -0.5)
    dy = n((T, d), 1.0)
    return x, wg, w_ug, w_down, dy


def gemm_flops(cfg, rows):
    d, f = cfg.d, cfg.f
    return {
        "gemm_fwd_upgate": 2.0 * rows * d * 2 * f,
        "gemm_fwd_down": 2.0 * rows * f * d,
        "gemm_bwd_dact": 2.0 * rows * d * f,
        "gemm_bwd_dx": 2.0 * rows * 2 * f * d,
        "gemm_wgrad_ug": 2.0 * rows * 2 * f * d,
        "gemm_wgrad_down": 2.0 * rows * d * f,
    }


def hbm_bytes(cfg):
    """Algorithmic HBM bytes per launch of the memory-bound kernels."""
    T, k, d, E = cfg.T, cfg.k, cfg.d, cfg.E
    return {
        "router_topk": T * d * 2 + d * E * 2 + T * k * 8 + 8 * E,
        "dispatch_permute": T * d * 2 + T * k * d * 2 + 8 * T * k,
        "combine": T * k * d * 2 + T * d * 2 + 8 * T * k,
        "combine_bwd": T * d * 2 + 2 * T * k * d * 2 + 8 * T * k,
        "router_bwd": T * k * d * 2 + T * d * 2 + 4 * T * k + T * d * 2,
        # fused peer-memory variants (ZP): the routed rows are also written to the owners' slots
        "dispatch_permute_p2p": T * d * 2 + 2 * T * k * d * 2 + 8 * T * k,
        "combine_bwd_p2p": T * d * 2 + 2 * T * k * d * 2 + 8 * T * k,
    }


def run_ours(args, ws, rank, local):
    from paper_2504_03871_b200 import ops
    from paper_2504_03871_b200.configs import CONFIGS, with_tokens
    from paper_2504_03871_b200.layer import moe_forward

    cfg = CONFIGS[args.config]
    if args.tokens:
        cfg = with_tokens(cfg, args.tokens)
    dev = torch.device("cuda", local)
    x, wg, w_ug, w_down, dy = make_layer_tensors(cfg, seed=1234 + rank, device=dev)
    params = [wg.requires_grad_(), w_ug.requires_grad_(), w_down.requires_grad_()]
    xg = x.requires_grad_()

    def step(x_in, dy_in):
        for p in params:
            p.grad = None
        x_in.grad = None
        xi = x_in
        y, idx = moe_forward(xi, params[0], params[1], params[2], cfg.k, args.max_ctas)
        y.backward(dy_in)
        return y

    # ---- warmup
    for _ in range(args.warmup):
        step(xg, dy)
    barrier(ws)

    # ---- timed region (device resident inputs)
    timer = ops.KernelTimer()
    ops.set_timer(timer)
    l0 = ops.LAUNCHES[0]
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier(ws)
        ev0.record(stream)
        for _ in range(args.steps):
            step(xg, dy)
        ev1.record(stream)
        barrier(ws)
    ops.set_timer(None)
    launches = (ops.LAUNCHES[0] - l0) // args.steps
    ms = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms, ws)
    ms_per_step = ms / args.steps
    tokens_total = cfg.T * ws * args.steps
    value = tokens_total / (ms / 1e3)

    # ---- per-kernel device durations inside the timed region
    summ = timer.summary()
    peaks = load_peaks()
    rows = cfg.T * cfg.k
    gf = gemm_flops(cfg, rows)
    gemm_ms = sum(summ[n][1] for n in gf if n in summ) / args.steps
    gemm_flop = sum(gf.values())
    gemm_tflops = gemm_flop / (gemm_ms / 1e3) / 1e12
    peak_t = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    kernels = {}
    for n, (cnt, tot) in summ.items():
        per = tot / cnt
        ent = {"launches_per_step": cnt // args.steps, "ms_per_launch": round(per, 4),
               "share_of_step": round(tot / ms_per_step / args.steps, 4) if ms_per_step else None}
        if n in gf:
            ent["tflops"] = round(gf[n] / (per / 1e3) / 1e12, 1)
            ent["frac_of_burst_peak"] = round(ent["tflops"] / peaks["bf16_tflops"], 3)
        hb = hbm_bytes(cfg)
        if n in hb:
            ent["gbs"] = round(hb[n] / (per / 1e3) / 1e9, 1)
            ent["frac_hbm"] = round(ent["gbs"] / peaks["hbm_gbs"], 3)
        kernels[n] = ent
    roofline = {
        "kernel": "grouped_gemm_kernel (K3: 6 tcgen05 GEMM launches per step)",
        "bound": "tensor",
        "achieved": round(gemm_tflops, 1),
        "peak": peak_t,
        "unit": "TFLOP/s",
        "frac": round(gemm_tflops / peak_t, 4),
        "frac_of_burst_peak": round(gemm_tflops / peaks["bf16_tflops"], 4),
        "frac_of_datasheet_2250": round(gemm_tflops / 2250.0, 4),
        "traffic": None,
        "traffic_algorithmic_bytes_per_step": gemm_min_bytes(cfg),
        "peak_source": peaks["source"] + ", sustained bf16 (kernel timed inside a long step)",
        "algorithmic_flops_per_step": gemm_flop,
        "gemm_ms_per_step": round(gemm_ms, 3),
    }

    tr = ncu_traffic(cfg.name, "grouped_gemm_kernel", 6)
    if tr is not None:
        roofline["traffic"] = tr["bytes"]
        roofline["traffic_unit"] = "bytes of DRAM read+write per step (the 6 K3 launches)"
        roofline["traffic_source"] = tr["source"]

    # ---- end-to-end through the public API with host buffers: every step copies its inputs
    # (x, dY) from pinned host memory and its results (the layer output y and the input gradient
    # dX) back to pinned host memory. The H2D copy of step i+1 runs on a copy stream under step
    # i's compute (double-buffered device inputs); the D2H copies of step i run on a second copy
    # stream under step i+1's compute. Everything is inside the timed region, which ends when the
    # last D2H copy has landed.
    x_host = x.detach().cpu().pin_memory()
    dy_host = dy.detach().cpu().pin_memory()
    y_host = [torch.empty(x_host.shape, dtype=x_host.dtype).pin_memory() for _ in range(2)]
    dx_host = [torch.empty(x_host.shape, dtype=x_host.dtype).pin_memory() for _ in range(2)]
    x_dev = [torch.empty_like(x.detach()) for _ in range(2)]
    dy_dev = [torch.empty_like(dy) for _ in range(2)]
    copy_stream = torch.cuda.Stream(dev)
    d2h_stream = torch.cuda.Stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]

    def h2d(i):
        b = i & 1
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[b])  # buffer b's previous step finished with it
            x_dev[b].copy_(x_host, non_blocking=True)
            dy_dev[b].copy_(dy_host, non_blocking=True)
            copied[b].record(copy_stream)

    e2e_warm = max(3, args.warmup)  # untimed pipelined steps (allocator and copy engines warm)
    e2e_last = e2e_warm + args.steps - 1

    def e2e_step(i):
        b = i & 1
        stream.wait_event(copied[b])
        if i < e2e_last:
            h2d(i + 1)
        xin = x_dev[b].detach().requires_grad_()
        for p in params:
            p.grad = None
        y, idx = moe_forward(xin, params[0], params[1], params[2], cfg.k, args.max_ctas)
        y.backward(dy_dev[b])
        consumed[b].record(stream)
        d2h_stream.wait_event(consumed[b])
        with torch.cuda.stream(d2h_stream):
            y.record_stream(d2h_stream)
            xin.grad.record_stream(d2h_stream)
            y_host[b].copy_(y.detach(), non_blocking=True)
            dx_host[b].copy_(xin.grad, non_blocking=True)

    for ev in consumed:
        ev.record(stream)
    h2d(0)
    for i in range(e2e_warm):  # warm-up of the pipelined path (the last one prefetches the first timed step)
        e2e_step(i)
    torch.cuda.synchronize()
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(e2e_warm, e2e_last + 1):
        e2e_step(i)
    stream.wait_stream(d2h_stream)  # the last step's results are on the host
    e1.record(stream)
    barrier(ws)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), ws)
    e2e = {"value": tokens_total / (e2e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": x_host.numel() * 2 + dy_host.numel() * 2,
           "d2h_bytes_per_step": y_host[0].numel() * 2 + dx_host[0].numel() * 2,
           "ms_per_step": round(e2e_ms / args.steps, 3),
           "note": "through moe_forward/backward: pinned H2D of each step's x and dY (prefetched one "
                   "step ahead on a copy stream) and pinned D2H of its y and dX (on a second copy "
                   "stream, overlapping the next step)"}

    out = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded randn inputs, random-init weights)",
        "config": {
            "workload": f"{cfg.name}: E={cfg.E} top-{cfg.k} d={cfg.d} f={cfg.f} T={cfg.T} tokens/GPU/step",
            "E": cfg.E, "k": cfg.k, "d_model": cfg.d, "d_ff": cfg.f, "tokens_per_gpu": cfg.T,
            "parallelism": "single GPU" if ws == 1 else f"{ws} data-parallel replicas",
            "l2": "inputs and weights (>3 GB) exceed the 126 MB L2; no flush",
        },
        "roofline": roofline,
        "kernels": kernels,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, args.cpu_baseline_tokens)
    if rank == 0:
        _emit(out)


def gemm_min_bytes(cfg) -> int:
    """Compulsory HBM bytes of the six K3 GEMMs of one step (every operand read once, every
    output written once): the floor roofline.traffic is compared with."""
    R, d, f, E = cfg.T * cfg.k, cfg.d, cfg.f, cfg.E
    x, h, act, w_ug, w_d = R * d * 2, R * 2 * f * 2, R * f * 2, E * 2 * f * d * 2, E * d * f * 2
    return ((x + w_ug + h + act)          # fwd up+gate (SwiGLU epilogue stores h and act)
            + (act + w_d + x)             # fwd down -> y
            + (x + w_d + h + h)           # bwd dact: dY, W_d, saved h -> dH
            + (h + w_ug + x)              # bwd dX
            + (h + x + w_ug)              # wgrad dW_ug
            + (x + act + w_d))            # wgrad dW_d


def ncu_traffic(config_name: str, kernel_prefix: str, launches: int):
    """DRAM bytes (read + write) of one step's launches of `kernel_prefix`, from the committed
    `ncu --set full` capture summary profiles/ncu_traffic_<config>.json (tools/summarize_ncu.py),
    or None when there is no capture for this config."""
    path = os.path.join(ROOT, "profiles", f"ncu_traffic_{config_name.split('-')[0]}.json")
    if not os.path.exists(path):
        return None
    rec = json.load(open(path))
    ls = [r for r in rec["launches"] if r["kernel"].startswith(kernel_prefix)][:launches]
    if len(ls) < launches or any(r["dram_read_bytes"] is None for r in ls):
        return None
    return {"bytes": int(sum(r["dram_read_bytes"] + r["dram_write_bytes"] for r in ls)),
            "source": os.path.relpath(path, ROOT) + " (" + rec["source"] + ")"}


def cpu_baseline(cfg, tokens: int):
    """The CPU oracle (fp32 PyTorch + numpy) on a bounded sample of the same layer."""
    from oracle import moe_oracle as orc
    from paper_2504_03871_b200.configs import make_inputs, with_tokens

    ncpu = os.cpu_count() or 1
    torch.set_num_threads(ncpu)
    c = with_tokens(cfg, tokens)
    inp = make_inputs(c, seed=0)
    from paper_2504_03871_b200.ops import interleave_gate_up

    w_ug = interleave_gate_up(inp.w_gate, inp.w_up)
    layer = orc.CpuLayer(inp.wg, w_ug, inp.w_down, c.k)  # fp32 parameters prepared once
    layer.step(inp.x, inp.dy)  # warm-up (thread pools, allocator)
    t0 = time.perf_counter()
    layer.step(inp.x, inp.dy)
    dt = time.perf_counter() - t0
    return {"value": tokens / dt, "unit": UNIT, "cores": ncpu, "kind": "port",
            "sample": f"{tokens} tokens of {cfg.name} (fwd+bwd, fp32 CPU oracle, {dt:.1f}s)"}


def stack_single_gpu(shape, layers: int, microbatches: int, dev, seed: int = 7,
                     chunk_tokens: int = 8192):
    """The ZP stack's work on ONE GPU with no pipeline (the scaling comparator for N > 1): the
    same tokens (microbatches x tokens_per_mb) and layers — pre-norm attention over the same
    tokens_per_mb-token sequences, then the MoE layer through the same native kernels — forward
    and backward, processed in chunks of `chunk_tokens` (8192: the bare layer's throughput there
    equals the N = 1 bench's at 16384, with half the activation memory) so each chunk's
    weight gradients are formed once per layer, like the ZP executor's (no per-micro-batch
    gradient read-modify-write; a chunk's gradients replace the previous chunk's). Returns
    MoE-layer tokens/s (tokens x layers / time), CUDA-event timed, one iteration after warm-up."""
    from paper_2504_03871_b200.executor import attention_block, rms_norm
    from paper_2504_03871_b200.layer import moe_forward

    g = torch.Generator(device=dev).manual_seed(seed)
    d, f, E, k, T = shape.d, shape.f, shape.E, shape.k, shape.tokens_per_mb
    heads = shape.heads or max(1, d // 128)
    total = T * microbatches
    C = max(T, (min(chunk_tokens, total) // T) * T)  # whole sequences per chunk

    def rnd(*sz, std=1.0):
        return (torch.randn(sz, generator=g, device=dev) * std).to(torch.bfloat16).requires_grad_()

    P = [dict(wqkv=rnd(d, 3 * d, std=d ** -0.5), wo=rnd(d, d, std=d ** -0.5), wg=rnd(d, E, std=d ** -0.5),
              w_ug=rnd(E, 2 * f, d, std=d ** -0.5), w_d=rnd(E, d, f, std=f ** -0.5)) for _ in range(layers)]
    x = [torch.randn((C, d), generator=g, device=dev).to(torch.bfloat16) for _ in range(2)]
    gy = [torch.randn((C, d), generator=g, device=dev).to(torch.bfloat16) for _ in range(2)]
    nchunks = (total + C - 1) // C

    def iteration():
        for j in range(nchunks):
            n = min(C, total - j * C)
            for p in P:
                for t in p.values():
                    t.grad = None
            h = x[j & 1][:n]
            for p in P:
                u = attention_block(h, p["wqkv"], p["wo"], heads, seq=T) if shape.attention else h * 1
                y, _ = moe_forward(rms_norm(u), p["wg"], p["w_ug"], p["w_d"], k)
                h = u + y
            h.backward(gy[j & 1][:n])

    iteration()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    iteration()
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    del P
    return total * layers / (ms / 1e3), ms


def run_zp(args, ws, rank, local):
    """N > 1: zebra-parallel stack of MoE transformer layers (C4 shape at 8 GPUs: 4 attention +
    4 expert ranks). value = MoE-layer tokens/s = tokens/iteration * layers / iteration time."""
    from paper_2504_03871_b200 import build_zp_graph, derive_task_durations
    from paper_2504_03871_b200 import ops
    from paper_2504_03871_b200.configs import CONFIGS
    from paper_2504_03871_b200.executor import (NativeBackend, ZpExecutor, ZpLayerShape, ZpP2PExecutor,
                                                execute)
    from paper_2504_03871_b200.planner import clamp_to_layer_capacity, make_zp_spec, plan_assignment
    from paper_2504_03871_b200.profiler import measure_durations
    from paper_2504_03871_b200.simulator import compute_metrics, validate_measured_timeline

    c = CONFIGS[args.config]
    M = args.attention_ranks or ws // 2
    N = ws - M
    if not 0 < M < ws or (M % N and N % M):
        raise SystemExit(f"--attention-ranks {M} of {ws}: need 0 < M < {ws} and M | N or N | M")
    dev = torch.device("cuda", local)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    caps = [float(v) for v in str(args.expert_capacity).split(",")]
    caps = caps * N if len(caps) == 1 else caps
    if len(caps) != N or min(caps) <= 0 or max(caps) > 1:
        raise SystemExit(f"--expert-capacity: need 1 or {N} weights in (0, 1], got {args.expert_capacity}")

    def ctas(w):  # capacity weight -> grouped-GEMM grid cap (0 = the whole GPU)
        return 0 if w >= 1.0 else int(math.ceil(w * sms))

    exp_ctas = ctas(caps[rank - M]) if rank >= M else 0
    hetero = len(set(caps)) > 1
    shape = ZpLayerShape(c.E, c.k, c.d, c.f, args.mb_tokens, attention=not args.no_attention,
                         router_skew=args.router_skew)
    # the per-GPU scaling comparator (rank 0): the identical stack on ONE GPU, measured first,
    # while the device holds nothing else (at 8 GPUs the ZP arena and activation pools alone take
    # ~100 GB per rank); every other rank waits at the barrier
    stack_ref = None
    if not args.no_stack_reference:
        if rank == 0:
            stack_ref = stack_single_gpu(shape, args.layers, M * args.microbatches, dev)
            torch.cuda.empty_cache()
            torch.cuda.reset_peak_memory_stats(dev)
        barrier(ws)
    loads = None
    if args.router_skew and not args.no_balanced_placement:
        # skewed router: expected per-expert loads (rank 0's measurement) drive a load-balanced
        # expert placement and the busiest-rank expert timing
        from paper_2504_03871_b200.profiler import measure_loads

        lt = torch.tensor(measure_loads(shape, device=dev), dtype=torch.int64, device=dev)  # noqa: E501
        dist.broadcast(lt, 0)
        loads = [int(v) for v in lt.tolist()]
    # the planner's expert GPU is the slowest expert rank (Algorithm 1 models one expert class)
    durs = measure_durations(shape, M, N, expert_max_ctas=ctas(min(caps)), device=dev, loads=loads,
                             capacity=caps if hetero else None, microbatches=args.microbatches,
                             balance_roles=not args.raw_attention_duration)
    # profiler -> planner, memory and transport: measured bytes per expert,
    # activation bytes per role and the device capacity become the spec's memory model (n_min /
    # n_max bounds of Algorithm 1); the (layer, micro-batch) exchange is timed on NCCL
    from paper_2504_03871_b200.executor import PeerArena
    from paper_2504_03871_b200.profiler import measure_exchange, measure_memory, memory_spec_fields

    memp = measure_memory(shape, device=dev)
    comm_ns = measure_exchange(M, N, args.mb_tokens, c.k, c.d)  # NCCL all-to-all of the rows
    # the exchange as the executor performs it with the chosen transport (a 1-layer, 1-micro-batch
    # run): the planner's dispatch / combine durations
    from paper_2504_03871_b200.profiler import measure_transport

    disp_groups = (dist.new_group(list(range(ws))), dist.new_group(list(range(ws))))
    tr = measure_transport(shape, M, N, NativeBackend(dev, max_ctas=exp_ctas if rank >= M else 0),
                           args.transport, *disp_groups)
    mt = torch.tensor([memp[k_] for k_ in sorted(memp)] + [comm_ns, tr["dispatch_ns"], tr["combine_ns"]],
                      dtype=torch.int64, device=dev)
    dist.broadcast(mt, 0)  # every rank plans with rank 0's probe
    memp = dict(zip(sorted(memp), (int(v) for v in mt[:-3].tolist())))
    comm_ns = int(mt[-3])
    transport_ns = {"dispatch_ns": int(mt[-2]), "combine_ns": int(mt[-1])}
    arena = PeerArena.bytes_needed(args.layers, args.microbatches, args.mb_tokens * M * c.k,
                                   args.mb_tokens * c.k, c.d) if args.transport == "p2p" else 0
    mem_fields = memory_spec_fields(memp, M, N, args.layers, args.microbatches, args.mb_tokens, c.k, arena)
    # every rank must plan identically: use rank 0's measurement
    t = torch.tensor([durs[k] for k in sorted(durs)], dtype=torch.int64, device=dev)
    dist.broadcast(t, 0)
    durs = dict(zip(sorted(durs), (int(v) for v in t.tolist())))
    from fractions import Fraction

    durs.update(transport_ns)
    from paper_2504_03871_b200.profiler import PLANNER_DURATION_KEYS

    plan_durs = {k_: v for k_, v in durs.items() if k_ in PLANNER_DURATION_KEYS}
    spec = make_zp_spec(M, N, args.layers, args.microbatches, c.E, c.k, args.mb_tokens, c.d,
                        asym_ea=not args.no_asym_ea, gamma=Fraction(durs["gamma_x100"], 100),
                        **plan_durs, **mem_fields)
    from paper_2504_03871_b200.costmodel import memory_bounds

    bounds = memory_bounds(spec)
    dur = derive_task_durations(spec)
    from paper_2504_03871_b200 import build_distep_graph

    clamped_layers = 0
    calibration = None
    if args.schedule == "distep":  # lockstep ablation (no cross-micro-batch overlap, no offload)
        graph = build_distep_graph(spec, dur)
        assignment = graph.assignment
    else:
        if args.offload:
            # explicit per-layer offload (the reference CLI's explicit plan, cli.py:93-106)
            from paper_2504_03871_b200 import ExpertAssignment

            assignment = ExpertAssignment(tuple(int(v) for v in args.offload.split(",")))
        else:
            assignment = plan_assignment(spec, dur)
            assignment, clamped_layers = clamp_to_layer_capacity(assignment, c.E, M, N)
            if (args.calibrate or args.router_skew > 0) and not args.no_calibrate and not args.no_asym_ea:
                # re-plan from durations measured inside a short pipeline run of this plan's
                # offloads (profiler.calibrate_in_pipeline): sustained clocks, real loads under skew
                from paper_2504_03871_b200.profiler import calibrate_in_pipeline

                offs = list(assignment.offload)
                cal_off = (min(offs), max(offs))
                cal = calibrate_in_pipeline(
                    shape, M, N, NativeBackend(dev, max_ctas=exp_ctas if rank >= M else args.attn_gemm_ctas),
                    cal_off, args.transport, *disp_groups, microbatches=args.microbatches,
                    expert_loads=loads, expert_capacity=caps if hetero else None, base=durs)
                keys = ("attn_fwd_ns", "expert_layer_fwd_ns", "single_expert_fwd_ns", "gamma_x100")
                ct = torch.tensor([cal[k_] for k_ in keys], dtype=torch.int64, device=dev)
                dist.broadcast(ct, 0)
                cal = dict(zip(keys, (int(v) for v in ct.tolist())))
                durs_cal = dict(durs, **cal)
                plan_cal = {k_: v for k_, v in durs_cal.items() if k_ in PLANNER_DURATION_KEYS}
                spec = make_zp_spec(M, N, args.layers, args.microbatches, c.E, c.k, args.mb_tokens, c.d,
                                    asym_ea=True, gamma=Fraction(durs_cal["gamma_x100"], 100),
                                    **plan_cal, **mem_fields)
                bounds = memory_bounds(spec)
                dur = derive_task_durations(spec)
                first = list(assignment.offload)
                assignment, clamped_layers = clamp_to_layer_capacity(plan_assignment(spec, dur), c.E, M, N)
                calibration = {"calibration_offload": list(cal_off), "durations_ns": cal,
                               "profiled_ns": {k_: durs[k_] for k_ in keys}, "offload_before": first,
                               "offload_after": list(assignment.offload)}
        graph = build_zp_graph(spec, dur, assignment, mode="zp-full")
    disp = dist.new_group(list(range(ws)))
    comb = dist.new_group(list(range(ws)))
    be = NativeBackend(dev, max_ctas=exp_ctas if rank >= M else args.attn_gemm_ctas,
                       comm_priority=args.comm_priority)
    ex_cls = ZpP2PExecutor if args.transport == "p2p" else ZpExecutor
    ex = ex_cls(graph, shape, M, N, rank, be, disp, comb, seed=1234, expert_loads=loads,
                expert_capacity=caps if hetero else None)
    for _ in range(args.warmup):
        ex.run()
    l0 = ops.LAUNCHES[0]
    barrier(ws)
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    timer = ops.KernelTimer()  # per-kernel device time, on each task's own stream
    ops.set_timer(timer)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            ex.run()
        ev1.record(stream)
        barrier(ws)
    ops.set_timer(None)
    ms = max_over_ranks(ev0.elapsed_time(ev1), ws)
    launches = (ops.LAUNCHES[0] - l0) // args.steps
    tokens_iter = args.mb_tokens * M * args.microbatches
    roofline, kernels = zp_roofline(timer.summary(), c, args, ws, rank, tokens_iter)
    e2e = zp_e2e(ex, args, ws, rank, dev, tokens_iter)
    tl = execute(graph, ex)  # one more iteration, measured per task
    hw = torch.tensor([ex.host_wait_s], device=dev)
    dist.all_reduce(hw, op=dist.ReduceOp.MAX)
    dl = bool(getattr(ex, "device_layout", False))
    pool = torch.tensor([float(getattr(ex, "pool_regrows", 0)), (ex.h_pool.numel() + ex.act_pool.numel() +
                         ex.dh_pool.numel()) * 2 / 2 ** 30 if dl else 0.0], device=dev)
    dist.all_reduce(pool, op=dist.ReduceOp.MAX)
    # peak device memory of the ZP run: per role (attention / expert ranks), max over ranks
    mem = torch.zeros(2, device=dev)
    mem[0 if rank < M else 1] = torch.cuda.max_memory_allocated(dev) / 2 ** 30
    dist.all_reduce(mem, op=dist.ReduceOp.MAX)
    value = tokens_iter * args.layers * args.steps / (ms / 1e3)
    if rank != 0:
        return
    met = compute_metrics(graph, tl, tokens_per_iteration=tokens_iter)
    viol = validate_measured_timeline(graph, tl)
    # measured mean duration per task kind on its home role vs the profiled (simulated) one
    kinds = {}
    for t in graph.tasks:
        ranks = range(0, M) if t.device == "attn" else range(M, ws)
        ds = [tl.per_rank[r][t.id][1] - tl.per_rank[r][t.id][0] for r in ranks if t.id in tl.per_rank[r]]
        if ds:
            k_ = kinds.setdefault(t.kind.value, [0.0, 0.0, 0])
            k_[0] += sum(ds) / len(ds)
            k_[1] += t.duration
            k_[2] += 1
    task_ms = {k: {"measured_ms": round(v[0] / v[2] / 1e6, 3), "simulated_ms": round(v[1] / v[2] / 1e6, 3)}
               for k, v in sorted(kinds.items())}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded randn inputs, random-init weights)",
        "config": {
            "workload": (f"{'ZP' if args.schedule == 'zp' else 'DistEP lockstep'} {M} attention + {N} expert ranks: {args.layers}-layer {c.name}-shaped MoE "
                         f"transformer stack, {args.microbatches} micro-batches x {args.mb_tokens} tokens per "
                         f"attention rank; value counts MoE-layer tokens (tokens x layers) per second"),
            "E": c.E, "k": c.k, "d_model": c.d, "d_ff": c.f, "layers": args.layers,
            "microbatches": args.microbatches, "tokens_per_microbatch": args.mb_tokens,
            "attention_block": not args.no_attention, "parallelism": f"zp{M}+{N}",
            "asym_ea_offload": list(assignment.offload),
            "asym_ea_layers_clamped_to_n_over_N": clamped_layers,
            "transport": args.transport, "schedule": args.schedule, "expert_capacity": caps,
            "comm_stream_priority": "high" if args.comm_priority else "default",
            "attention_rank_gemm_ctas": args.attn_gemm_ctas or sms,
            "expert_grid_ctas": [ctas(w) or sms for w in caps],
            "router_skew_zipf": args.router_skew,
            "expert_placement": ("contiguous" if loads is None and not hetero else
                                 "load-balanced (LPT over measured loads / capacity weights)"),
            "memory_probe_bytes": memp,
            "memory_bounds": {"n_min": bounds.n_min, "n_max": bounds.n_max,
                              "expert_mem": mem_fields["expert_mem"],
                              "non_expert_mem_attention": mem_fields["non_expert_mem_attention"],
                              "non_expert_mem_expert": mem_fields["non_expert_mem_expert"],
                              "capacity": mem_fields["exp_capacity"]},
            "measured_exchange_ns": {"nccl_all_to_all": comm_ns, "executor_transport": transport_ns},
            "expert_loads_per_mb": loads,
            "measured_durations_ns": durs,
            "l2": "activations and weights exceed the 126 MB L2; no flush",
        },
        "zp": {
            "measured_makespan_ms": tl.makespan / 1e6,
            "simulated_makespan_ms": None,
            "attn_utilization": float(met.devices["attn"].utilization_of_makespan),
            "exp_utilization": float(met.devices["exp"].utilization_of_makespan),
            "timeline_violations": len(viol),
            "task_durations": task_ms,
        },
        "roofline": roofline,
        "kernels": kernels,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    from paper_2504_03871_b200 import simulate, default_orders

    if stack_ref is not None:
        # the same work (all M x R micro-batches, all layers, attention + MoE) on this one GPU
        # without the pipeline: the per-GPU comparator for scaling (the N = 1 bench line is the
        # bare MoE layer, BASELINE configs[1])
        v1, ms1 = stack_ref
        out["scaling_reference"] = {
            "value": v1, "unit": UNIT, "ms_per_iteration": round(ms1, 3),
            "workload": ("identical stack and token count on ONE GPU, no pipeline, in 8192-token chunks "
                         "(weight gradients formed once per chunk and layer, as the "
                         "executor forms them once per layer) — rank 0, before the ZP setup"),
            "per_gpu_efficiency": value / (ws * v1),
        }
    out["zp"]["simulated_makespan_ms"] = simulate(graph, default_orders(graph)).makespan / 1e6
    # planning cost per iteration (host, pure Python, bit-identical to the reference's zpsim):
    # Algorithm 1 + graph construction + stream orders + list-scheduling simulation. It runs once
    # per plan, off the per-iteration critical path; reported to show it is negligible.
    tp0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        if args.schedule == "distep":
            g_ = build_distep_graph(spec, dur)
        else:
            a_ = plan_assignment(spec, dur) if not args.offload else assignment
            g_ = build_zp_graph(spec, dur, clamp_to_layer_capacity(a_, c.E, M, N)[0], mode="zp-full")
        simulate(g_, default_orders(g_))
    out["zp"]["planning_ms"] = round((time.perf_counter() - tp0) / reps * 1e3, 3)
    out["zp"]["planning_tasks"] = len(graph.tasks)
    if calibration is not None:
        out["zp"]["calibration"] = calibration
    # the same schedule replayed with each compute task at its measured duration (slowest rank
    # of its role): what the executor would reach with no issue stalls (communication tasks
    # keep their planned time)
    import dataclasses

    from paper_2504_03871_b200.taskgraph import TaskGraph

    comm = {"DispF", "CombF", "DispB", "CombB"}
    newt = []
    for t in graph.tasks:
        ranks = range(0, M) if t.device == "attn" else range(M, ws)
        ds = [tl.per_rank[r][t.id][1] - tl.per_rank[r][t.id][0] for r in ranks if t.id in tl.per_rank[r]]
        dur = t.duration if (t.kind.value in comm or not ds) else max(ds)  # slowest rank of the role
        newt.append(dataclasses.replace(t, duration=dur))
    g2 = TaskGraph(graph.mode, graph.layers, graph.microbatches, tuple(newt), graph.edges,
                   graph.assignment, graph.forward_only)
    out["zp"]["resimulated_makespan_ms"] = simulate(g2, default_orders(g2)).makespan / 1e6
    out["zp"]["host_count_wait_ms_max_rank"] = round(float(hw) * 1e3, 3)
    out["zp"]["receive_layout"] = ({"where": "device (hm_zp_layout)", "pool_factor": getattr(ex, "pool_factor", None),
                                    "pool_regrows_max_rank": int(pool[0]), "pool_gib_max_rank": round(float(pool[1]), 2)}
                                   if dl else {"where": "host"})
    out["zp"]["peak_mem_gib"] = {"attention_ranks": round(float(mem[0]), 1),
                                 "expert_ranks": round(float(mem[1]), 1),
                                 "rank0_zp_run": round(torch.cuda.max_memory_allocated(dev) / 2 ** 30, 1)}
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(c, args.cpu_baseline_tokens)
    _emit(out)


GEMM_NAMES = ("gemm_fwd_upgate", "gemm_fwd_down", "gemm_fwd_down_p2p", "gemm_bwd_dact", "gemm_bwd_dx",
              "gemm_bwd_dx_p2p", "gemm_wgrad_ug", "gemm_wgrad_down")


def zp_roofline(summ, c, args, ws, rank, tokens_iter):
    """N > 1: K3 (every rank's grouped-GEMM launches) against the sustained tensor peak, and the
    attention-side HBM kernels of rank 0. `summ` is this rank's KernelTimer summary over the
    timed steps (CUDA events on each launch's own stream). Collective: every rank calls it."""
    peaks = load_peaks()
    gemm_ms = sum(summ[n][1] for n in GEMM_NAMES if n in summ)
    t = torch.tensor([gemm_ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)  # sum of K3 device time over all ranks
    flop = 18.0 * tokens_iter * c.k * c.d * c.f * args.layers * args.steps  # fwd 6 + bwd 12 per row
    per_gpu = flop / (float(t) / 1e3) / 1e12 if float(t) > 0 else 0.0
    peak_t = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    roofline = {
        "kernel": "grouped_gemm_kernel (K3) on every rank: expert ranks' experts and the Asym-EA "
                  "offloaded experts on attention ranks",
        "bound": "tensor", "achieved": round(per_gpu, 1), "peak": peak_t, "unit": "TFLOP/s",
        "frac": round(per_gpu / peak_t, 4),
        "frac_of_burst_peak": round(per_gpu / peaks["bf16_tflops"], 4),
        "traffic": None,
        "achieved_definition": "algorithmic FLOP of all K3 launches of the job (18*tokens*k*d*f per "
                               "layer) / the sum over ranks of their K3 device time: the per-GPU "
                               "rate while K3 runs",
        "peak_source": peaks["source"] + ", sustained bf16",
        "gemm_ms_per_step_all_ranks": round(float(t) / args.steps, 3),
    }
    kernels = {}
    if rank == 0:
        from paper_2504_03871_b200.configs import with_tokens

        hb = hbm_bytes(with_tokens(c, args.mb_tokens))
        for n, (cnt, tot) in summ.items():
            per = tot / cnt
            ent = {"launches_per_step": cnt // args.steps, "ms_per_launch": round(per, 4)}
            if n in hb:
                ent["gbs"] = round(hb[n] / (per / 1e3) / 1e9, 1)
                ent["frac_hbm"] = round(ent["gbs"] / peaks["hbm_gbs"], 3)
            kernels[n] = ent
        kernels["_note"] = "rank 0 (an attention rank); per-launch device time of each native op"
    return roofline, kernels


def zp_e2e(ex, args, ws, rank, dev, tokens_iter):
    """N > 1 end to end through the executor: every iteration the attention ranks copy each
    micro-batch's input and output gradient from pinned host memory into the executor's input
    buffers (H2D) and read each micro-batch's input gradient back (D2H), all inside the timed
    region; time = max over ranks. Collective."""
    ex.keep_input_grads = True
    hin = {j: t.detach().cpu().pin_memory() for j, t in ex.inputs.items()}
    hgo = {j: t.detach().cpu().pin_memory() for j, t in ex.out_grads.items()}
    hdx = {j: torch.empty(t.shape, dtype=t.dtype).pin_memory() for j, t in ex.inputs.items()}
    stream = torch.cuda.current_stream()

    def iteration():
        for j in hin:
            ex.inputs[j].copy_(hin[j], non_blocking=True)
            ex.out_grads[j].copy_(hgo[j], non_blocking=True)
        ex.run()
        for j in hdx:
            hdx[j].copy_(ex.input_grads[j], non_blocking=True)

    iteration()
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        iteration()
    e1.record(stream)
    barrier(ws)
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    ex.keep_input_grads = False
    nb = torch.tensor([sum(t.numel() * 2 for t in hin.values()) * 2, sum(t.numel() * 2 for t in hdx.values())],
                      dtype=torch.int64, device="cuda")
    dist.all_reduce(nb)  # whole-job bytes per step (attention ranks hold the batches)
    return {"value": tokens_iter * args.layers * args.steps / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": int(nb[0]), "d2h_bytes_per_step": int(nb[1]),
            "ms_per_step": round(ms / args.steps, 3),
            "note": "through ZpExecutor.run(): per iteration, pinned H2D of every micro-batch's input "
                    "and output gradient and pinned D2H of its input gradient on the attention "
                    "ranks (bytes summed over ranks)"}


def run_reference(args, ws, rank):
    """Reference arm: the CPU oracle port of the layer (the reference has no MoE layer code;
    SURVEY F3) on the host cores, each step a bounded token sample of the same config."""
    if rank != 0:
        return
    from oracle import moe_oracle as orc
    from paper_2504_03871_b200.configs import CONFIGS, make_inputs, with_tokens
    from paper_2504_03871_b200.ops import interleave_gate_up

    cfg = CONFIGS[args.config]
    ncpu = os.cpu_count() or 1
    torch.set_num_threads(ncpu)
    c = with_tokens(cfg, args.cpu_tokens)
    inp = make_inputs(c, seed=0)
    w_ug = interleave_gate_up(inp.w_gate, inp.w_up)
    layer = orc.CpuLayer(inp.wg, w_ug, inp.w_down, c.k)  # fp32 parameters prepared once
    for _ in range(max(args.warmup, 1)):
        layer.step(inp.x, inp.dy)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        layer.step(inp.x, inp.dy)
    dt = time.perf_counter() - t0
    value = c.T * args.steps / dt
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded)", "impl": "reference",
        "config": {"workload": f"{cfg.name}: E={cfg.E} top-{cfg.k} d={cfg.d} f={cfg.f}; "
                               f"each step a {c.T}-token sample on the host CPU"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ncpu, "kind": "port",
                         "sample": f"{c.T} tokens per step, fp32 CPU oracle fwd+bwd"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    _emit(out)


_OUT = sys.stdout


def relaunch(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-run this command under torch.distributed.run
    with N ranks on this node (one per GPU, rendezvous on 127.0.0.1). Rank 0's JSON line reaches
    our stdout unchanged; returns the launcher's exit code."""
    import socket
    import subprocess

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def _plain(obj, path="$"):
    """JSON-ready copy of obj; a stray tensor is converted and reported on stderr with its path."""
    if isinstance(obj, dict):
        return {k: _plain(v, f"{path}.{k}") for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_plain(v, f"{path}[{i}]") for i, v in enumerate(obj)]
    if isinstance(obj, torch.Tensor):
        print(f"bench.py: tensor at {path} in the result line", file=sys.stderr)
        return obj.tolist()
    return obj


def _emit(obj) -> None:
    """Print the one JSON result line on the original stdout."""
    _OUT.write(json.dumps(_plain(obj)) + "\n")
    _OUT.flush()


def main():
    global _OUT
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # native libraries (NCCL) may print banners on fd 1; keep fd 1 for stderr and write the
        # JSON line to a duplicate of the original stdout
        _OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3"])
    ap.add_argument("--tokens", type=int, default=0, help="override tokens per GPU per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--cpu-tokens", type=int, default=2048, help="tokens per --impl reference step")
    ap.add_argument("--cpu-baseline-tokens", type=int, default=2048)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layers", type=int, default=8, help="ZP (N>1): MoE transformer layers")
    ap.add_argument("--microbatches", type=int, default=8, help="ZP (N>1): micro-batches R")
    ap.add_argument("--mb-tokens", type=int, default=4096, help="ZP (N>1): tokens per micro-batch per attention rank")
    ap.add_argument("--attention-ranks", type=int, default=0,
                    help="ZP: attention ranks M (default half the ranks, e.g. 4 + 4 at 8 GPUs; 6 gives BASELINE C5's "
                         "6 + 2, 3 the 3 + 1 analogue at 4 GPUs)")
    ap.add_argument("--no-attention", action="store_true", help="ZP: identity attention block")
    ap.add_argument("--attn-gemm-ctas", type=int, default=0,
                    help="ZP: cap the offloaded-expert GEMM grid on attention ranks (SMs left to the comm kernels)")
    ap.add_argument("--comm-priority", action="store_true", help="ZP: high stream priority for the comm lanes")
    ap.add_argument("--raw-attention-duration", action="store_true",
                    help="ZP: plan with the attention forward as measured (no fwd+bwd role normalisation)")
    ap.add_argument("--no-asym-ea", action="store_true", help="ZP: keep all experts on expert ranks")
    ap.add_argument("--calibrate", action="store_true",
                    help="ZP: re-plan Asym-EA from durations measured inside a short pipeline run "
                         "(on by default with --router-skew > 0)")
    ap.add_argument("--no-calibrate", action="store_true", help="ZP: never re-plan from the pipeline run")
    ap.add_argument("--router-skew", type=float, default=0.0,
                    help="ZP: Zipf exponent of a per-expert router bias (skewed expert loads)")
    ap.add_argument("--no-balanced-placement", action="store_true",
                    help="ZP with --router-skew: keep the contiguous expert placement")
    ap.add_argument("--no-stack-reference", action="store_true",
                    help="ZP: skip the single-GPU run of the same stack (scaling comparator)")
    ap.add_argument("--schedule", default="zp", choices=["zp", "distep"],
                    help="ZP: zebra-parallel schedule, or the DistEP lockstep ablation")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="ZP: NVLink peer-memory transport fused into the kernels, or NCCL send/recv")
    ap.add_argument("--offload", default="",
                    help="ZP: explicit experts offloaded per expert rank, per layer (e.g. 2,2,2,2,2,2,2,2) "
                         "instead of the Asym-EA plan")
    ap.add_argument("--expert-capacity", default="1.0",
                    help="ZP: capacity weight of the expert ranks, one value or one per expert rank "
                         "(e.g. 1,0.5); grouped-GEMM grid = ceil(w*SMs) on that rank")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if ws_env != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}")
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    ws, rank, local = dist_setup() if args.impl == "ours" else (
        int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if ws > 1:
        run_zp(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
