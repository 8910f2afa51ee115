#!/usr/bin/env python3
"""Write tests/golden/verify_4e18_windows.json by running the CPU ORACLE only:
aggregates, histogram and the SHA-256 of the per-n p_min dump (u32 little-endian,
index (n - lo_e)/2) of windows of config C5's range [4e18 - 1e11, 4e18)
(BASELINE.json configs[4]).

Windows: the top and the bottom of the range (they hold the SURVEY Appendix A
golden points and window maxima 3191 / 2311 / 2293 / 3167) and two seeded
interior windows.  Nothing here touches the CUDA path.

usage: python scripts/make_golden_4e18.py [--evens 2097152] [--threads N]
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle  # noqa: E402

TOP = 4 * 10**18
BOT = TOP - 10**11
SEED = 20260302


def windows(evens):
    span = 2 * evens
    rng = np.random.default_rng(SEED)
    w = [(TOP - span, TOP), (BOT, BOT + span)]
    for _ in range(2):
        lo = BOT + 2 * int(rng.integers(0, (10**11 - span) // 2))
        w.append((lo, lo + span + 2 * int(rng.integers(0, 100)) + 1))   # ragged tail
    return w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--evens", type=int, default=1 << 22)
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    a = ap.parse_args()
    out = {"source": "oracle/gb_oracle.c via scripts/make_golden_4e18.py (CPU oracle only)",
           "p_fast": 65521, "chk_def": "chk = sum n*p_min(n) mod 2^64 (SURVEY.md 8(b)); chk192 = sum p_min(n)*floor(n/192) mod 2^64",
           "dump_hash": "sha256 of the u32 little-endian per-n dump", "windows": []}
    for lo, hi in windows(a.evens):
        t0 = time.time()
        r, d = oracle.verify(lo, hi, p_fast=65521, threads=a.threads, dump=True)
        res = {k: int(r[k]) for k in oracle.FIELDS}
        res["hist"] = {str(i): int(c) for i, c in enumerate(r["hist"]) if c}
        out["windows"].append({"lo": lo, "hi": hi, "result": res,
                               "dump_sha256": hashlib.sha256(d.astype("<u4").tobytes()).hexdigest(),
                               "oracle_seconds": round(time.time() - t0, 1)})
        print(lo, hi, res["max_pmin"], res["max_pmin_n"], f"{time.time() - t0:.1f}s", flush=True)
    path = os.path.join(ROOT, "tests", "golden", "verify_4e18_windows.json")
    json.dump(out, open(path, "w"), indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
