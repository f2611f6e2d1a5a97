"""Generate tests/golden/schedule_golden.json from the REFERENCE itself (zpsim, imported from a
temporary copy of /root/reference/pkg/src so nothing is written into the read-only mount).

    python tests/golden/gen_golden.py            # needs /root/reference (this container only)

The GPU box never runs this; it only reads the committed JSON.
"""

from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile
import types

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import schedule_cases as sc  # noqa: E402

REF = os.environ.get("HETERMOE_REFERENCE", "/root/reference")


def import_reference():
    """Import zpsim from a scratch copy; returns the api namespace used by record()."""
    sys.dont_write_bytecode = True
    tmp = tempfile.mkdtemp(prefix="zpsim_ref_")
    shutil.copytree(os.path.join(REF, "pkg", "src", "zpsim"), os.path.join(tmp, "zpsim"))
    sys.path.insert(0, tmp)
    import zpsim  # noqa: F401
    from zpsim import core, costmodel, planner, scheduler, simulator, taskgraph

    return api_from(core, costmodel, taskgraph, scheduler, simulator, planner)


def api_from(core, costmodel, taskgraph, scheduler, simulator, planner):
    ns = types.SimpleNamespace()
    for mod, names in (
        (core, ["parse_config", "spec_to_config", "ExpertAssignment"]),
        (costmodel, ["derive_task_durations", "workload_shape", "routed_tokens_per_microbatch",
                     "memory_bounds", "MemoryBounds"]),
        (taskgraph, ["offload_scaling", "token_flow", "build_zp_graph", "graph_to_json",
                     "build_distep_graph"]),
        (scheduler, ["chunk_sizes", "asym_ea_offload", "compute_l_busy", "bubble_ledger",
                     "default_orders", "OffloadPlanInputs"]),
        (simulator, ["simulate", "compute_metrics", "bubble_intervals", "export_trace",
                     "load_trace_intervals", "validate_timeline"]),
        (planner, ["tokens_per_iteration", "offload_inputs"]),
    ):
        for n in names:
            setattr(ns, n, getattr(mod, n))
    return ns


def offload_cases(seed: int = 7):
    """Direct Algorithm-1 inputs (exact rationals), including bound / infeasible corners."""
    import random
    from fractions import Fraction

    rng = random.Random(seed)
    cases = []
    for _ in range(300):
        M = rng.choice([1, 2, 4, 3, 6, 8])
        N = rng.choice([1, 2, 4, 3, 6, 8])
        if M % N and N % M:
            continue
        per = rng.choice([1, 2, 3, 4, 6])
        cases.append({
            "experts_per_layer": N * per, "layers": rng.randint(1, 12), "attention_gpus": M,
            "expert_gpus": N,
            "attn_fwd": f"{rng.randint(0, 5000)}/{rng.choice([1, 1, 3, 7])}",
            "single_expert_on_attn": f"{rng.randint(0, 5000)}/{rng.choice([1, 2])}",
            "expert_layer_on_expert": f"{rng.randint(0, 9000)}/{rng.choice([1, 1, 5])}",
            "n_min": rng.choice([0, 0, 0, 1, 2, 5, 9]),
            "n_max": rng.choice([None, None, 0, 1, 3, 8, 20]),
            "squeeze_mode": rng.choice(["verbatim", "rederived"]),
        })
    return cases


def offload_record(api, case):
    from fractions import Fraction

    kw = dict(case)
    for key in ("attn_fwd", "single_expert_on_attn", "expert_layer_on_expert"):
        kw[key] = Fraction(kw[key])
    try:
        plan = api.asym_ea_offload(api.OffloadPlanInputs(**kw))
    except Exception as exc:  # noqa: BLE001
        return {"error": type(exc).__name__}
    return sc._plan_rec(plan)


def main():
    api = import_reference()
    cases = [(name, cfg) for name, cfg in sc.reference_configs(REF)]
    cases += [(f"random{i}", cfg) for i, cfg in enumerate(sc.random_configs(60))]
    out = {"generator": "tests/golden/gen_golden.py (zpsim reference)", "cases": []}
    for name, cfg in cases:
        out["cases"].append({"name": name, "config": cfg, "record": sc.record(api, cfg)})
    out["offload"] = [{"inputs": c, "record": offload_record(api, c)} for c in offload_cases()]
    path = os.path.join(HERE, "schedule_golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
        fh.write("\n")
    print(f"wrote {path}: {len(out['cases'])} configs, {len(out['offload'])} offload cases")


if __name__ == "__main__":
    main()
