"""Markdown table of the ZP sweep JSON lines (tools/zp_sweep.sh)."""
import glob
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep"
rows = []
for p in sorted(glob.glob(os.path.join(d, "*.json"))):
    try:
        j = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception:
        continue
    c, z = j["config"], j["zp"]
    rows.append((j["n_gpus"], os.path.basename(p)[:-5], j["value"], z["measured_makespan_ms"],
                 z["simulated_makespan_ms"], z.get("resimulated_makespan_ms"), c["asym_ea_offload"],
                 c.get("transport"), c.get("schedule", "zp"), c["router_skew_zipf"], c["expert_capacity"],
                 j["clocks"].get("sm_mhz")))
print("| GPUs | run | layer-tokens/s | measured ms | simulated ms | resimulated ms | offload o_l | transport | schedule | Zipf α | capacity w | SM MHz |")
print("|---:|---|---:|---:|---:|---:|---|---|---|---:|---:|---:|")
for r in sorted(rows, key=lambda r: (r[0], r[1])):
    print(f"| {r[0]} | {r[1]} | {r[2]:,.0f} | {r[3]:.1f} | {r[4]:.1f} | {r[5]:.1f} | {r[6]} | {r[7]} | {r[8]} | {r[9]} | {r[10]} | {r[11]} |")
