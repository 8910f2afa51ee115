#!/usr/bin/env python3
"""Write tests/golden/verify_<N>.json by running the CPU ORACLE only.

Results over disjoint ranges compose (counts and hist add, max_pmin takes the
max with the smallest n, first_unresolved_n the min, chk adds mod 2^64), so the
range [4, N] is computed in pieces of `--piece-chunks` chunks and each finished piece
is appended to a resumable JSONL cache.  Pieces are whole chunks of CHUNK_EVENS
evens counted from the range's first even, and the oracle's per-chunk
chk = sum n * p_min mod 2^64 goes to tests/golden/chk_<tag>.npy (uint64, one per
chunk) so a GPU run can be compared piece by piece through its per-n dumps.
Nothing here touches the CUDA path: every stored value comes from oracle/ (see
the oracle's header for citations).

usage: python scripts/make_golden.py --N 1e12 [--threads 6] [--piece-chunks 298]
       python scripts/make_golden.py --window c5   (the 4e18 window)
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle  # noqa: E402

U64 = (1 << 64) - 1
CHUNK_EVENS = 1 << 24
CHK_DEF = "chk = sum n*p_min(n) mod 2^64 (SURVEY.md 8(b))"


def merge(a, b):
    if a is None:
        return dict(b)
    out = dict(a)
    for k in ("evens", "verified", "fastpath_unresolved", "unresolved", "sum_pmin"):
        out[k] = a[k] + b[k]
    out["chk"] = (a["chk"] + b["chk"]) & U64
    out["first_unresolved_n"] = min(a["first_unresolved_n"], b["first_unresolved_n"])
    if (b["max_pmin"], -b["max_pmin_n"]) > (a["max_pmin"], -a["max_pmin_n"]):
        out["max_pmin"], out["max_pmin_n"] = b["max_pmin"], b["max_pmin_n"]
    h = dict(a["hist"])
    for i, c in b["hist"].items():
        h[i] = h.get(i, 0) + c
    out["hist"] = h
    return out


def to_json_result(r):
    d = {k: r[k] for k in oracle.FIELDS}
    d["hist"] = {str(i): int(c) for i, c in enumerate(r["hist"]) if c}
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=float, default=None, help="the range [4, N]")
    ap.add_argument("--window", choices=["c5"], default=None,
                    help="c5: [4e18 - 1e11, 4e18) (BASELINE.json configs[4])")
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    ap.add_argument("--piece-chunks", type=int, default=298,
                    help="chunks of 2^24 evens per oracle call (298 -> 1e10 integers)")
    ap.add_argument("--p-fast", type=int, default=65521)
    args = ap.parse_args()
    piece = 2 * CHUNK_EVENS * args.piece_chunks
    if args.window == "c5":
        LO, HI, tag = 4 * 10**18 - 10**11, 4 * 10**18, "c5_4e18"
    else:
        N = int(args.N)
        LO, HI, tag = 4, N + 1, f"{N:.0e}".replace("+", "")
    assert LO % 2 == 0
    cache = os.path.join(ROOT, "tests", "golden", f".cache2_verify_{tag}.jsonl")
    outp = os.path.join(ROOT, "tests", "golden", f"verify_{tag}.json")
    done = {}
    if os.path.exists(cache):
        with open(cache) as f:
            for line in f:
                rec = json.loads(line)
                done[(rec["lo"], rec["hi"])] = rec
    total = None
    chunks = []
    t_all = 0.0
    lo = LO
    while lo < HI:
        hi = min(lo + piece, HI)
        if (lo, hi) not in done:
            t0 = time.time()
            r, _ = oracle.verify(lo, hi, p_fast=args.p_fast, threads=args.threads,
                                 chunk_evens=CHUNK_EVENS)
            dt = time.time() - t0
            rec = {"lo": lo, "hi": hi, "seconds": dt, "threads": args.threads,
                   "result": to_json_result(r), "chunk_chk": [int(x) for x in r["chunk_chk"]]}
            with open(cache, "a") as f:
                f.write(json.dumps(rec) + "\n")
            done[(lo, hi)] = rec
            print(f"[{lo}, {hi}) {dt:.1f}s", flush=True)
        rec = done[(lo, hi)]
        t_all += rec["seconds"]
        res = dict(rec["result"])
        res["hist"] = {int(k): v for k, v in res["hist"].items()}
        total = merge(total, res)
        chunks.extend(rec["chunk_chk"])
        lo = hi
    total["hist"] = {str(k): v for k, v in sorted(total["hist"].items())}
    assert (sum(chunks) & U64) == total["chk"]
    np.save(os.path.join(ROOT, "tests", "golden", f"chk_{tag}.npy"), np.array(chunks, dtype=np.uint64))
    doc = {"lo": LO, "hi": HI, "p_fast": args.p_fast,
           "chk_def": CHK_DEF, "chunk_evens": CHUNK_EVENS, "chunk_chk_file": f"chk_{tag}.npy",
           "source": "oracle/gb_oracle.c via scripts/make_golden.py (CPU oracle only)",
           "oracle_seconds": round(t_all, 1), "result": total}
    with open(outp, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", outp)


if __name__ == "__main__":
    main()
