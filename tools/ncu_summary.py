"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel (share of time)."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID") + 1
    hdr = rows[start - 1]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    lines = [f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:40s} {n:8d} {t:12.1f} {100 * t / tot:6.1f}%")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
