#!/usr/bin/env python3
"""Per-region breakdown of an ncu --set full --import-source capture of verify_kernel:
warp instructions, stall samples and the top stall reasons per source region of
gb_verify.cu (regions = function line ranges, found by name in the source).

usage: python scripts/ncu_regions.py gpurun_out/<capture>.ncu-rep"""
import csv
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2603_02621_b200", "csrc", "gb_verify.cu")
# (region, regex of the first line of the function or block that starts it)
MARKS = [
    ("sieve:helpers", r"^template <bool DEF_TILE>\s*$"),
    ("sieve:clear_bit", r"^__device__ __forceinline__ void clear_bit"),
    ("sieve:medium progression", r"^__device__ __forceinline__ void mark_progression2"),
    ("sieve:carry policy", r"^__device__ __forceinline__ uint64_t carry_policy"),
    ("sieve:window (tiny patterns)", r"^__device__ __forceinline__ void sieve6_window\("),
    ("sieve:medium setup", r"^\s*// medium primes \(31 < p"),
    ("sieve:medium warp loop", r"^\s*// one warp per medium prime"),
    ("sieve:steady large", r"^\s*// large primes: one thread per prime"),
    ("acc", r"^struct CtaAcc"),
    ("mark:mark_step", r"^struct Lane6"),
    ("mark:hist8", r"^// Per-warp counts of 8 candidates"),
    ("mark:block8", r"^__device__ __forceinline__ void block8\("),
    ("mark:phase1q", r"^// ---- phase 1 with kW words per lane"),
    ("mark:phase1r", r"^// ---- phase 1b"),
    ("mark:phase2", r"^// phase 2: candidates"),
    ("mark:replay", r"^// max p_min among the unrolled hits"),
    ("mark:finish_word", r"^// candidates past the unrolled tables"),
    ("mark:valid/special", r"^__device__ __forceinline__ uint32_t valid_mask"),
    ("steady_count", r"^// Steady primes of the window starting"),
    ("mark:ClassWork", r"^struct ClassWork"),
    ("mark:round_q", r"^\s*// one phase-1 round: words"),
    ("mark:stage", r"^\s*// candidates \[kC1, kP1\) for cnt staged"),
    ("mark:round/mark_tile", r"^\s*static __device__ __forceinline__ void round\("),
    ("flush_hist", r"^// shared histograms -> result vector"),
    ("kernel body", r"^// UNROLL: every unrolled candidate"),
    ("sieve_out", r"^// gb_sieve_segment: tiles"),
]


def regions():
    lines = open(SRC).read().splitlines()
    starts = []
    for name, rx in MARKS:
        for i, l in enumerate(lines, 1):
            if re.search(rx, l):
                starts.append((i, name))
                break
    starts.sort()
    return starts


def region_of(starts, ln):
    cur = "header"
    for s, n in starts:
        if ln >= s:
            cur = n
    return cur


def breakdown(rep):
    """{region: {"ins", "samp", "stall": {...}}} of one capture"""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    starts = regions()
    agg, names, f = {}, None, None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            f = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            names = r
            continue
        if r[0] == "" or names is None:
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        key = region_of(starts, ln) if f == "gb_verify.cu" else ("intrinsics" if f.endswith(".hpp") else f)
        d = agg.setdefault(key, {"ins": 0, "samp": 0, "stall": {}})
        num = lambda x: int(x) if x.isdigit() else 0
        d["ins"] += num(r[7])
        d["samp"] += num(r[4])
        for i, n in enumerate(names):
            if n.startswith("stall_") and "(Not Issued)" not in n:
                d["stall"][n[6:]] = d["stall"].get(n[6:], 0) + num(r[i])
    return agg


def phase_shares(rep):
    """share of stall samples (~ time) and of warp instructions in the sieve regions,
    the marking regions and the rest"""
    agg = breakdown(rep)
    ts = sum(d["samp"] for d in agg.values()) or 1
    ti = sum(d["ins"] for d in agg.values()) or 1
    out = {"samples": {}, "instructions": {}}
    for k, d in agg.items():
        ph = "sieve" if k.startswith("sieve") else ("mark" if k.startswith("mark") or k in ("acc", "flush_hist")
                                                     else "other")
        out["samples"][ph] = out["samples"].get(ph, 0) + d["samp"] / ts
        out["instructions"][ph] = out["instructions"].get(ph, 0) + d["ins"] / ti
    return out


def main():
    rep = sys.argv[1]
    agg = breakdown(rep)
    ti = sum(d["ins"] for d in agg.values()) or 1
    ts = sum(d["samp"] for d in agg.values()) or 1
    print(f"total warp instructions {ti:,}  stall samples {ts:,}")
    print(f"{'region':32s} {'instr%':>7s} {'samp%':>7s}  top stalls")
    for k, d in sorted(agg.items(), key=lambda x: -x[1]["samp"]):
        st = d["stall"]
        tot = sum(st.values()) or 1
        top = sorted(st.items(), key=lambda x: -x[1])[:4]
        print(f"{k:32s} {100 * d['ins'] / ti:7.2f} {100 * d['samp'] / ts:7.2f}  " +
              " ".join(f"{n} {100 * v / tot:.0f}%" for n, v in top))


if __name__ == "__main__":
    main()
