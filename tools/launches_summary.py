"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel name."""
import csv
import sys
from collections import defaultdict


def summarise(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(d["Metric Unit"], 1e-6)
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
    tot = sum(t for _, t in agg.values())
    out = [f"{'kernel':44s} {'launches':>8s} {'total ms':>10s} {'ms/launch':>10s} {'share':>6s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:44s} {n:8d} {t:10.3f} {t / n:10.4f} {t / tot:6.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
