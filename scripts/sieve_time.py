#!/usr/bin/env python3
"""Time gb_sieve_segment (K-SIEVE standalone) over the top 2^34 integers of [4, N]:
median of 10 launches, GB/s of odd bitset written.  usage: python scripts/sieve_time.py [--N 1e12]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_02621_b200.verifier import Verifier  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=float, default=1e12)
a = ap.parse_args()
N = int(a.N)
v = Verifier(hi_max=N + 1, origin=max(0, N + 1 - 2**40) & ~1)
w_hi = (N - 3) // 128
w_lo = w_hi - (1 << 27)
out = torch.empty(w_hi - w_lo, dtype=torch.int64, device=v.device)
for _ in range(2):
    v.sieve_segment(w_lo, w_hi - w_lo)
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    from paper_2603_02621_b200 import gb
    gb.gb_sieve_segment(v.ctx, w_lo, w_hi - w_lo, out, v.stream)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
h = int(out.sum().item()) & 0xFFFFFFFF
print(f"SIEVE lib={os.environ.get('GB_LIB', 'default')} N={N:.0e} median_ms={ts[5]:.3f} "
      f"GB/s={8 * (w_hi - w_lo) / ts[5] / 1e6:.1f} digest={h}")
