"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel name,
count, total and mean device time and share of the listed time."""
import csv
import sys
from collections import defaultdict


def main(path, title=""):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    units = set()
    for r in rows[1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki]
        if len(name) > 70:
            name = name[:67] + "..."
        v = float(r[vi].replace(",", ""))
        units.add(r[ui])
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v for _, v in agg.values())
    print(f"# {title}  units: {sorted(units)}; cold-cache, serialised: compare SHARES")
    print(f"{'kernel':72s} {'n':>5s} {'total':>14s} {'mean':>11s} {'share':>7s}")
    for name, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:72s} {n:5d} {v:14.1f} {v / n:11.1f} {v / tot:7.4f}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
