#!/usr/bin/env python3
"""Summarise an ncu report (read here, no GPU) into profiles/<name>.json + .md:
duration, IPC, pipe utilisation, stall mix, DRAM/L2/shared traffic, and the
instruction mix by phase of verify_kernel.

usage: python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_verify --evens 1073741824
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

KEYS = {
    "gpu__time_duration.sum": "duration",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "pipe_xu_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "pipe_lsu_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def ncu(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_base(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
             "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}
    return float(v) * scale.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--evens", type=float, default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = ncu(a.rep, "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    res = {"report": a.rep, "kernel": vals[hdr.index("Kernel Name")], "note": a.note}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            try:
                res[name] = to_base(vals[i].replace(",", ""), units[i])
            except ValueError:
                res[name] = vals[i]
    src = ncu(a.rep, "source", ["--print-source", "sass"])
    shdr, data = src[1], src[2:]
    stalls = [h for h in shdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = defaultdict(int)
    for r in data:
        for h in stalls:
            tot[h[6:]] += int(r[shdr.index(h)] or 0)
    T = sum(tot.values()) or 1
    res["stall_pct"] = {k: round(100 * v / T, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]}
    if "verify_kernel" in res["kernel"]:
        # sieve vs marking share of the kernel (stall samples ~ time), for bench.py's
        # separate K-SIEVE / K-MARK rooflines
        import os
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from ncu_regions import phase_shares
        sh = phase_shares(a.rep)
        res["phase_share_samples"] = {k: round(v, 4) for k, v in sh["samples"].items()}
        res["phase_share_instructions"] = {k: round(v, 4) for k, v in sh["instructions"].items()}
    if a.evens:
        res["evens"] = a.evens
        res["evens_per_s_under_ncu"] = a.evens / res["duration"]
        res["warp_instr_per_even"] = res.get("warp_instructions", 0) / a.evens
        res["dram_bytes_per_even"] = (res.get("dram_read", 0) + res.get("dram_write", 0)) / a.evens
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as f:
        f.write(f"# ncu summary: {res['kernel'][:80]}\n\n{a.note}\n\n| metric | value |\n|---|---|\n")
        for k, v in res.items():
            if k in ("stall_pct", "kernel", "note", "report") or isinstance(v, dict):
                continue
            f.write(f"| {k} | {v:.6g} |\n" if isinstance(v, float) else f"| {k} | {v} |\n")
        for k in ("phase_share_samples", "phase_share_instructions"):
            if k in res:
                f.write(f"| {k} | " + ", ".join(f"{n} {v:.3f}" for n, v in res[k].items()) + " |\n")
        f.write("\nStall mix (% of warp-state samples): " +
                ", ".join(f"{k} {v}" for k, v in res["stall_pct"].items()) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
