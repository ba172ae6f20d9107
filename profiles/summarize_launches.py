"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", "")) * {"ns": 1, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(r[ui], 1)
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    out = [f"total kernel time {tot / 1e6:.3f} ms over {sum(n for n, _ in agg.values())} launches",
           f"{'kernel':52s} {'launches':>8s} {'ms':>9s} {'share':>7s} {'avg us':>9s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k[:52]:52s} {n:8d} {t / 1e6:9.3f} {100 * t / tot:6.1f}% {t / n / 1e3:9.2f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
