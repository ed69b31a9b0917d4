"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV):
per-kernel launch count, total / mean device time and share of the total."""
import csv
import io
import sys
from collections import defaultdict


def main(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v *= {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'mean ms':>9s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {n:8d} {t:10.3f} {t / n:9.4f} {100 * t / tot:6.2f}%")
    print(f"{'total':40s} {sum(v[0] for v in agg.values()):8d} {tot:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
