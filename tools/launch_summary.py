"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel count, total, share."""
import csv
import re
import sys
from collections import defaultdict


def summarise(path, top=15):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v *= {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
        name = re.sub(r"\(.*", "", r["Kernel Name"])
        rows.append((name, v))
    agg = defaultdict(lambda: [0, 0.0])
    for n, v in rows:
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v for _, v in rows)
    print(f"{path}: {len(rows)} launches, {tot / 1e3:.2f} ms total")
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"  {v / 1e3:9.3f} ms {100 * v / tot:5.1f}%  x{c:<6d} {n[:90]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summarise(p)
