#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum]
--csv` launch list by kernel: launches, total / average duration, share of the
listed time and (when captured) average DRAM bytes per launch.

usage: tools/ncu_summary.py launches.csv "command description" > profiles/<name>.txt
"""
import collections
import csv
import sys

SCALE_T = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
SCALE_B = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path: str, title: str) -> None:
    rows = list(csv.reader(open(path, errors="replace")))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, ii = hdr.index("Kernel Name"), hdr.index("ID")
    mi, ui, vi = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    launches = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        key = r[ii]
        name = r[ki].split("(")[0].replace("hpsb::", "").replace("<unnamed>::", "").strip()
        name = name.split("<")[0] if name.startswith("void ") is False else name
        d = launches.setdefault(key, {"name": name, "us": 0.0, "bytes": 0.0})
        val = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            d["us"] += val * SCALE_T.get(r[ui], 1.0)
        elif r[mi].startswith("dram__bytes"):
            d["bytes"] += val * SCALE_B.get(r[ui], 1.0)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in launches.values():
        a = agg[d["name"]]
        a[0] += 1
        a[1] += d["us"]
        a[2] += d["bytes"]
    tot = sum(v[1] for v in agg.values())
    print(f"ncu launch list: {title}")
    print("serialised launches (no PDL overlap): compare shares, not absolute times")
    print(f"{'kernel':40s} {'launches':>8s} {'total_us':>11s} {'avg_us':>9s} {'share':>7s} {'MB/launch':>10s} {'GB/s':>8s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {n:8d} {t:11.1f} {t / n:9.2f} {100 * t / tot:6.1f}% {b / n / 1e6:10.3f} "
              f"{(b / (t * 1e-6) / 1e9 if t else 0):8.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
