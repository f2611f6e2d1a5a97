"""Summarise an `ncu --csv --metrics ...` launch list: one row per launch, one column per metric
(`python tools/ncu_csv.py file.csv [file2.csv ...]`)."""
import csv
import sys


def rows(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    out = {}
    for r in csv.DictReader(lines):
        key = (int(r["ID"]), r["Kernel Name"].split("(")[0].replace("void ", ""))
        out.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return out


def main():
    for path in sys.argv[1:]:
        print(path)
        tot = {}
        for (i, name), m in sorted(rows(path).items()):
            cells = "  ".join(f"{k.split('__')[1].split('.')[0]}={v / 1e9:.3f}G" if "bytes" in k
                              else f"{k.split('__')[1].split('.')[0]}={v / 1e6:.3f}ms" for k, v in sorted(m.items()))
            print(f"  {i:3d} {name[:60]:60s} {cells}")
            for k, v in m.items():
                tot[k] = tot.get(k, 0.0) + v
        print("  total", "  ".join(f"{k}={v:.4g}" for k, v in sorted(tot.items())))


if __name__ == "__main__":
    main()
