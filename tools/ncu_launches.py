#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, total, share."""
import collections
import csv
import re
import sys


def kname(full: str) -> str:
    s = full.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    s = re.sub(r"^void\s+", "", s)
    m = re.match(r"([\w:]+(?:<[^()]*>)?)", s)
    return m.group(1) if m else s[:60]


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= mi or r[0] == "ID":
            continue
        v = float(r[mi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        a = agg[kname(r[ki])]
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:44s} {v[0]:8d} {v[1]:10.1f} {v[1] / v[0]:9.2f} {v[1] / tot:6.3f}")
    print(f"{'TOTAL':44s} {sum(v[0] for v in agg.values()):8d} {tot:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
