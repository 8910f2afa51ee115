#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total ns, share of the GPU time.  Read here, no GPU.

usage: python scripts/launch_list.py gpurun_out/launches_c4.csv "<title>" > profiles/<name>.md"""
import csv
import sys
from collections import defaultdict


def main():
    path, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0])
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        a = agg[r[ki]]
        a[0] += 1
        a[1] += int(float(r[vi].replace(",", "")))
    tot = sum(v[1] for v in agg.values()) or 1
    print(f"# Launch list: {title}\n")
    print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised; "
          "shares, not absolute times, compare with the live run)\n")
    print("| kernel | launches | total ns | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k[:70]} | {n} | {t} | {100 * t / tot:.3f}% |")


if __name__ == "__main__":
    main()
