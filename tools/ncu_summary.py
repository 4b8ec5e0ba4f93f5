#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel.

usage: tools/ncu_summary.py launches.csv "command description" > profiles/<name>.txt
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path: str, title: str) -> None:
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0].replace("hpsb::", "").replace("<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    print(f"ncu --metrics gpu__time_duration.sum --clock-control none: {title}")
    print("cold-cache, serialised launches: compare shares, not absolute times")
    print(f"{'kernel':44s} {'launches':>8s} {'total_us':>11s} {'avg_us':>9s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:44s} {n:8d} {t:11.1f} {t / n:9.2f} {100 * t / tot:6.1f}%")
    print(f"{'total':44s} {sum(v[0] for v in agg.values()):8d} {tot:11.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
