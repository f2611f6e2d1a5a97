"""Shared case generator + record function for schedule / Asym-EA parity.

``record(api, config)`` runs the planning API of either the reference (``zpsim``) or this
package on one config dict and returns a JSON-able summary (exact integers, Fractions as
"p/q" strings, sha256 digests of the large structures). ``gen_golden.py`` stores the
reference's records; ``tests/test_schedule_parity.py`` recomputes them with
``paper_2504_03871_b200`` and requires equality.
"""

from __future__ import annotations

import copy
import hashlib
import json
import os
import random
import tempfile
from fractions import Fraction

REF_CONFIGS = ("minimal.json", "short_seq_offload.json", "heterogeneous_sweep.json")


def fr(x):
    if isinstance(x, Fraction):
        return f"{x.numerator}/{x.denominator}"
    if isinstance(x, float):
        return repr(x)
    return x


def digest(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True, default=str).encode()).hexdigest()[:24]


def _lanes_key(orders):
    return {f"{k[0]}/{k[1]}": list(v) for k, v in sorted(orders.items())}


def _timeline_rec(api, graph, tl, tokens):
    m = api.compute_metrics(graph, tl, tokens_per_iteration=tokens, steady_window=(1, graph.layers))
    dev = {}
    for name, d in sorted(m.devices.items()):
        dev[name] = [d.busy, d.first_start, d.last_end, d.bubble_total, d.drain_wait,
                     fr(d.utilization), fr(d.utilization_of_makespan)]
    starts = [tl.starts[t.id] for t in graph.tasks]
    ends = [tl.ends[t.id] for t in graph.tasks]
    bubbles = {f"{k[0]}/{k[1]}": api.bubble_intervals(graph, tl, k) for k in sorted(tl.lanes)}
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "trace.json")
        api.export_trace(graph, tl, p)
        with open(p, "rb") as fh:
            trace_sha = hashlib.sha256(fh.read()).hexdigest()[:24]
        intervals = api.load_trace_intervals(p)
    return {
        "makespan": tl.makespan,
        "timeline": digest([starts, ends]),
        "violations": api.validate_timeline(graph, tl),
        "metrics": [m.iteration_time, fr(m.throughput_tokens_per_ns), dev, fr(m.steady_state_utilization)],
        "bubbles": digest(bubbles),
        "trace_file": trace_sha,
        "trace_intervals": digest(sorted((list(k), list(v)) for k, v in intervals.items())),
    }


def _graph_rec(api, spec, durations, assignment, mode, backward):
    try:
        g = api.build_zp_graph(spec, durations, assignment=assignment, mode=mode, include_backward=backward)
    except Exception as exc:  # noqa: BLE001
        return {"error": type(exc).__name__}
    gj = api.graph_to_json(g)
    orders = api.default_orders(g)
    tl = api.simulate(g, orders)
    out = {
        "ntasks": len(g.tasks),
        "nedges": len(g.edges),
        "graph": digest(gj),
        "orders": digest(_lanes_key(orders)),
        "order_lens": {f"{k[0]}/{k[1]}": len(v) for k, v in sorted(orders.items())},
    }
    out.update(_timeline_rec(api, g, tl, api.tokens_per_iteration(spec)))
    if len(g.tasks) <= 40:
        out["graph_full"] = gj
        out["orders_full"] = _lanes_key(orders)
        out["starts"] = [tl.starts[t.id] for t in g.tasks]
    return out


def _plan_rec(plan):
    return {"assignment": list(plan.assignment.offload), "chunk": list(plan.chunk),
            "t_gather": fr(plan.t_gather), "t_squeeze": fr(plan.t_squeeze), "alpha": fr(plan.alpha),
            "beta": fr(plan.beta), "residuals": [fr(r) for r in plan.residuals], "note": plan.note}


def record(api, config: dict) -> dict:
    """Everything the planning layer computes for one config."""
    try:
        spec = api.parse_config(copy.deepcopy(config))
    except Exception as exc:  # noqa: BLE001
        return {"parse_error": type(exc).__name__,
                "violations": len(getattr(exc, "violations", []) or [])}
    rec = {"roundtrip": api.parse_config(api.spec_to_config(spec)) == spec}
    dur = api.derive_task_durations(spec)
    rec["durations"] = [dur.attn_fwd, dur.expert_layer_fwd_on_expert_gpu,
                        dur.single_expert_fwd_on_attn_gpu, dur.dispatch, dur.combine,
                        fr(dur.backward_factor)]
    sh = api.workload_shape(spec)
    rec["shape"] = [sh.tokens_per_microbatch_per_attn_gpu, fr(sh.tokens_per_expert_gpu), sh.seq_len]
    rec["routed"] = api.routed_tokens_per_microbatch(spec)
    rec["tokens_per_iteration"] = api.tokens_per_iteration(spec)
    try:
        b = api.memory_bounds(spec)
        rec["bounds"] = [b.n_min, b.n_max]
    except Exception as exc:  # noqa: BLE001
        rec["bounds"] = type(exc).__name__
        b = None
    L = spec.model.layers
    assignments = {"zeros": api.ExpertAssignment.zeros(L)}
    M, N = spec.cluster.attention_gpus, spec.cluster.expert_gpus
    nested = M % N == 0 or N % M == 0
    if nested:
        rec["chunk"] = list(api.chunk_sizes(M, N))
        try:
            inputs = api.offload_inputs(spec, dur, b) if b is not None else api.offload_inputs(
                spec, dur, api.MemoryBounds(0, None))
            plan = api.asym_ea_offload(inputs)
            rec["plan"] = _plan_rec(plan)
            assignments["plan"] = plan.assignment
            rec["l_busy"] = fr(api.compute_l_busy(inputs.expert_layer_on_expert, inputs.attn_fwd))
            rec["ledger"] = [fr(x) for x in api.bubble_ledger(inputs)]
        except Exception as exc:  # noqa: BLE001
            rec["plan"] = type(exc).__name__
    if spec.run.offload is not None:
        assignments["explicit"] = api.ExpertAssignment(spec.run.offload)
    graphs = {}
    for aname, a in assignments.items():
        try:
            sc, shr = api.offload_scaling(spec, a)
            rec[f"scaling_{aname}"] = [[fr(x) for x in sc], [fr(x) for x in shr]]
            rec[f"flow_{aname}"] = [
                {k: fr(v) for k, v in api.token_flow(spec, a, l).items()} for l in range(1, L + 1)]
        except Exception as exc:  # noqa: BLE001
            rec[f"scaling_{aname}"] = type(exc).__name__
        for mode in ("zp-full", "zp-theorem"):
            for bwd in (True, False):
                graphs[f"{aname}|{mode}|{int(bwd)}"] = _graph_rec(api, spec, dur, a, mode, bwd)
    rec["graphs"] = graphs
    try:
        dg = api.build_distep_graph(spec, dur)
        dtl = api.simulate(dg, api.default_orders(dg))
        rec["distep"] = [len(dg.tasks), digest([list(e) for e in dg.edges]), dtl.makespan,
                         digest(_lanes_key(api.default_orders(dg)))]
    except Exception as exc:  # noqa: BLE001
        rec["distep"] = type(exc).__name__
    return rec


# ---------------------------------------------------------------------------------------------
# case generation


def base_config(M=1, N=1, L=3, R=3, n=6, k=2, tables=True, seed=0) -> dict:
    cfg = {
        "cluster": {"attention_gpus": M, "expert_gpus": N, "link_bandwidth": 100_000_000_000,
                    "bytes_per_token": 4096},
        "model": {"layers": L, "experts_per_layer": n, "top_k": k, "hidden_dim": 64,
                  "seq_len": 4096, "microbatches": R, "sequences_per_microbatch": 1,
                  "expert_mem": 0, "activation_mem_per_token": 0},
        "profile": {},
        "run": {"mode": "zp-full", "gamma": 2.0, "seed": seed},
    }
    if tables:
        cfg["profile"] = {
            "attention_gpu": {"name": "fast", "memory_capacity": 10**12,
                              "durations": {"attn_fwd": 3000, "single_expert_fwd": 3000}},
            "expert_gpu": {"name": "slow", "memory_capacity": 10**12,
                           "durations": {"expert_layer_fwd": 4000}},
            "comm": {"dispatch": 0, "combine": 0},
        }
    else:
        cfg["profile"] = {
            "attention_gpu": {"name": "fast", "memory_capacity": 48 * 2**30,
                              "coefficients": {"attn_linear": 50, "attn_quadratic": 0.003, "expert": 120}},
            "expert_gpu": {"name": "slow", "memory_capacity": 16 * 2**30,
                           "coefficients": {"attn_linear": 60, "attn_quadratic": 0.03, "expert": 150}},
            "non_expert_mem_attention": 2 * 2**30,
            "non_expert_mem_expert": 2**30,
        }
    return cfg


def random_configs(count: int, seed: int = 20261018):
    rng = random.Random(seed)
    out = []
    for i in range(count):
        M = rng.choice([1, 1, 2, 2, 4, 3, 6])
        N = rng.choice([1, 2, 2, 4, 3, 8])
        per = rng.choice([1, 2, 3, 4, 6])
        n = N * per
        L = rng.randint(1, 6)
        R = rng.randint(1, 5)
        tables = rng.random() < 0.6
        cfg = base_config(M, N, L, R, n, min(rng.choice([1, 2, 2, 4]), n), tables, seed=i)
        cfg["run"]["mode"] = rng.choice(["zp-full", "zp-full", "zp-theorem"])
        cfg["run"]["gamma"] = rng.choice([1.0, 2.0, 1.5, 3])
        cfg["run"]["squeeze"] = rng.choice(["verbatim", "rederived"])
        if tables:
            a = rng.randint(1, 9000)
            cfg["profile"]["attention_gpu"]["durations"] = {
                "attn_fwd": a, "single_expert_fwd": rng.choice([a, rng.randint(1, 9000), 1234.5])}
            cfg["profile"]["expert_gpu"]["durations"] = {
                "expert_layer_fwd": rng.choice([a, a + rng.randint(1, 5000), rng.randint(1, 9000)])}
            cfg["profile"]["comm"] = {"dispatch": rng.choice([0, 0, 7, 250]),
                                      "combine": rng.choice([0, 3, 250.5])}
        else:
            cfg["model"]["seq_len"] = rng.choice([512, 4096, 8192, 16384])
            cfg["model"]["expert_mem"] = rng.choice([0, 157286400, 3 * 2**30])
            cfg["model"]["activation_mem_per_token"] = rng.choice([0, 4096])
            cfg["cluster"]["link_bandwidth"] = rng.choice([10**11, 4 * 10**11])
        if rng.random() < 0.4 and cfg["run"]["mode"] == "zp-full":
            cfg["run"]["asym_ea"] = True
        if rng.random() < 0.25:
            n2 = (M // N) if M % N == 0 else 1
            cfg["run"]["offload"] = [rng.choice([0, n2, 2 * n2]) for _ in range(L)]
        if rng.random() < 0.05:
            cfg["model"]["top_k"] = n + 1  # invalid on purpose
        if rng.random() < 0.05:
            cfg["cluster"]["bogus"] = 1  # unknown key -> ConfigError
        out.append(cfg)
    return out


def reference_configs(ref_root: str):
    out = []
    for name in REF_CONFIGS:
        with open(os.path.join(ref_root, "pkg", "configs", name)) as fh:
            out.append((name, json.load(fh)))
    return out
