#!/usr/bin/env python3
"""One short launch of each libgb kernel for ncu (keeps replays cheap):
gb_verify_range over the top 2^span integers of [4, N] (or of [lo, hi) with --hi)
and gb_sieve_segment over a window of the same size.
usage: python scripts/prof_one.py [--N 1e12] [--span 32] [--hi 4e18 --lo-window 3999999900000000000]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2603_02621_b200.verifier import Verifier  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=float, default=1e12)
ap.add_argument("--hi", type=int, default=None, help="exclusive top of the range (default N + 1)")
ap.add_argument("--origin", type=int, default=None)
ap.add_argument("--span", type=int, default=32)
ap.add_argument("--p-max", type=int, default=65521)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--time", type=int, default=0, help="time this many verify launches (after 2 warm-ups)")
a = ap.parse_args()
HI = a.hi if a.hi is not None else int(a.N) + 1
lo = HI - (1 << a.span)
v = Verifier(hi_max=HI, p_max=a.p_max, origin=a.origin if a.origin is not None else max(0, lo) & ~1)
r = v.new_result()
for _ in range(a.reps):
    v.verify(lo, HI, r)
v.finalize(r)
w = v.sieve_segment((lo - 3) // 128, (1 << a.span) // 128 - 2)
torch.cuda.synchronize()
d = v.decode(r)
print({k: d[k] for k in ("evens", "verified", "fastpath_unresolved", "max_pmin", "max_pmin_n", "sum_pmin")})
if a.time:
    r2 = v.new_result()
    for _ in range(2):
        v.verify(lo, HI, r2)
    ts = []
    for _ in range(a.time):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        v.verify(lo, HI, r2)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ev = d["evens"]
    print(f"TIME lib={os.environ.get('GB_LIB', 'default')} median_ms={ts[len(ts)//2]:.3f} "
          f"min_ms={ts[0]:.3f} evens_per_s={ev / (ts[len(ts)//2] / 1e3):.4e}")
