"""Planning cost per plan (host, single thread): the reference zpsim (imported from a scratch
copy of /root/reference — this container only) next to this package's bit-identical
reimplementation, on the C4 shape (4 attention + 4 expert ranks, L = R = 8) with B200-measured
durations. Both produce the same makespan; prints one JSON line.

    python tools/planning_cost.py > profiles/r1_planning_cost.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from gen_golden import api_from, import_reference  # noqa: E402

from paper_2504_03871_b200 import core, costmodel, planner, scheduler, simulator, taskgraph  # noqa: E402
from paper_2504_03871_b200.planner import make_zp_spec  # noqa: E402


def plan_and_simulate(api, spec):
    dur = api.derive_task_durations(spec)
    b = api.memory_bounds(spec)
    plan = api.asym_ea_offload(api.offload_inputs(spec, dur, b))
    g = api.build_zp_graph(spec, dur, plan.assignment, mode="zp-full")
    tl = api.simulate(g, api.default_orders(g))
    return len(g.tasks), tl.makespan, list(plan.assignment.offload)


def best_of(fn, reps=5):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), out


def main():
    ours = api_from(core, costmodel, taskgraph, scheduler, simulator, planner)
    ref = import_reference()
    # profiled B200 durations of the C2-shaped ZP layer (profiles/r1_zp4_final.json)
    spec = make_zp_spec(4, 4, 8, 8, 8, 2, 4096, 4096, attn_fwd_ns=585900, expert_layer_fwd_ns=2121484,
                        single_expert_fwd_ns=2117337, dispatch_ns=87154, combine_ns=87154, asym_ea=True)
    ref_spec = ref.parse_config(ours.spec_to_config(spec))
    t_ref, r_ref = best_of(lambda: plan_and_simulate(ref, ref_spec))
    t_our, r_our = best_of(lambda: plan_and_simulate(ours, spec))
    assert r_ref == r_our, (r_ref, r_our)
    print(json.dumps({
        "what": "Algorithm 1 + build_zp_graph + default_orders + simulate, C4 shape (M=N=4, L=R=8), one plan",
        "tasks": r_our[0], "makespan_ns": r_our[1], "offload": r_our[2],
        "reference_zpsim_ms": round(t_ref * 1e3, 2), "this_package_ms": round(t_our * 1e3, 2),
        "threads": 1, "host": os.uname().machine,
    }))


if __name__ == "__main__":
    main()
