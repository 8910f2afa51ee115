#!/usr/bin/env python3
"""Per-source-line view of an ncu report (needs -lineinfo): warp instructions
executed and stall samples per CUDA line, plus sums over named line ranges
(phases of verify_kernel).  Read here, no GPU.

usage: python scripts/ncu_lines.py gpurun_out/prof.ncu-rep [--top 40] [--ranges sieve=188-426,mark=428-1000]
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--ranges", default="")
    ap.add_argument("--file", default="gb_verify.cu")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr = None, None
    per = defaultdict(lambda: [0, 0, ""])      # (file, line) -> [inst, samples, text]
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0]:
            continue
        ie = hdr.index("Instructions Executed")
        sm = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            inst = int(r[ie] or 0)
            samp = int(r[sm] or 0)
        except ValueError:
            continue
        e = per[(fname, int(r[0]))]
        e[0] += inst
        e[1] += samp
        e[2] = r[1][:90]
    tot_i = sum(v[0] for v in per.values()) or 1
    tot_s = sum(v[1] for v in per.values()) or 1
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s}")
    for (f, ln), (i, s, t) in sorted(per.items(), key=lambda x: -x[1][1])[:a.top]:
        print(f"{f}:{ln:5d}  inst {100 * i / tot_i:5.1f}%  samples {100 * s / tot_s:5.1f}%  {t}")
    if a.ranges:
        print()
        for spec in a.ranges.split(","):
            name, rng = spec.split("=")
            lo, hi = map(int, rng.split("-"))
            i = sum(v[0] for (f, ln), v in per.items() if f == a.file and lo <= ln <= hi)
            s = sum(v[1] for (f, ln), v in per.items() if f == a.file and lo <= ln <= hi)
            print(f"{name:12s} lines {lo}-{hi}: inst {100 * i / tot_i:5.1f}%  samples {100 * s / tot_s:5.1f}%")
        for f in sorted({f for f, _ in per}):
            i = sum(v[0] for (ff, _), v in per.items() if ff == f)
            s = sum(v[1] for (ff, _), v in per.items() if ff == f)
            print(f"file {f:20s} inst {100 * i / tot_i:5.1f}%  samples {100 * s / tot_s:5.1f}%")


if __name__ == "__main__":
    main()
