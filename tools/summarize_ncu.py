"""Summarise ncu outputs into profiles/ (run here, on the CPU box, on files from gpurun_out/).

  python tools/summarize_ncu.py launches <launches.csv> <out.md> [--step-kernels N]
  python tools/summarize_ncu.py full <report.ncu-rep> <out.md>
"""

import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor smem-read active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem throughput %"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors (tex)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_dim_x", "cluster x"),
    ("launch__registers_per_thread", "regs/thread"),
]


def _short(name: str) -> str:
    m = re.match(r"(?:void )?(?:\w+::)*(\w+)(<[^()]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def launches(path, out):
    text = open(path).read()
    body = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(body)))
    agg = OrderedDict()
    total = 0.0
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = _short(r["Kernel Name"])
        v = float(r["Metric Value"]) / 1e3  # ns -> us
        n, s = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, s + v)
        total += v
    lines = [f"# ncu launch list summary: `{path}`", "",
             "Cold-cache, serialised per-launch times (compare SHARES, not absolutes).", "",
             "| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
    for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {s:.1f} | {s / total:.3f} |")
    lines.append(f"| **total** | {sum(n for n, _ in agg.values())} | {total:.1f} | 1.000 |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary: `{path}`", "",
             "| kernel | " + " | ".join(lbl for _, lbl in FULL_METRICS) + " |",
             "|---|" + "---:|" * len(FULL_METRICS)]
    for r in data:
        cells = []
        for m, _ in FULL_METRICS:
            if m in idx:
                u = units[idx[m]]
                cells.append(f"{r[idx[m]]} {u}".strip())
            else:
                cells.append("n/a")
        lines.append(f"| `{_short(r[idx['Kernel Name']])}` | " + " | ".join(cells) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    # JSON sidecar: per-launch DRAM bytes (bench.py reads it for roofline.traffic)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}

    def val(r, m, table):
        i = idx.get(m)
        if i is None or not r[i]:
            return None
        return float(r[i].replace(",", "")) * table.get(units[i], 1.0)

    recs = [{"kernel": _short(r[idx["Kernel Name"]]),
             "dram_read_bytes": val(r, "dram__bytes_read.sum", scale),
             "dram_write_bytes": val(r, "dram__bytes_write.sum", scale),
             "duration_s": val(r, "gpu__time_duration.sum", tscale)} for r in data]
    json.dump({"source": path, "launches": recs}, open(os.path.splitext(out)[0] + ".json", "w"), indent=1)


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    (launches if mode == "launches" else full)(src, dst)
