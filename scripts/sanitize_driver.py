#!/usr/bin/env python3
"""Small invocations of every libgb kernel for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck), each checked against the CPU oracle so a
sanitizer run is also a parity run.  SURVEY.md section 8(c), test T-sanitize.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_driver.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2603_02621_b200.verifier import Verifier  # noqa: E402


def check(got, want, what):
    for k in oracle.AGG_FIELDS:
        assert got[k] == want[k], (what, k, got[k], want[k])


# C1-sized ranges: K-BASE, the fused verify kernel (with dump), fallback, sieve-out, per-n
v = Verifier(hi_max=10**6 + 1, p_max=65521)
for lo, hi, p in ((4, 2 * 10**5 + 1, 65521), (4, 5 * 10**4, 5), (999000, 10**6 + 1, 97)):
    got, d = v.run(lo, hi, p_max=p, dump=True)
    want, wd = oracle.verify(lo, hi, p_fast=p, dump=True)
    assert np.array_equal(d.cpu().numpy().astype(np.uint32), wd)
    check(got, want, (lo, hi, p))
    got, _ = v.run(lo, hi, p_max=p, mode="pern")
    check(got, want, ("pern", lo, hi, p))
w = v.sieve_segment(0, 64).cpu().numpy().view(np.uint64)
ob = oracle.sieve_window(3, 3 + 128 * 64)
assert np.array_equal(w, np.packbits(ob, bitorder="little").view(np.uint64))
# NEXT-4 partition counts and NEXT-3 single_check
c = v.partition_counts(4, 20001).cpu().numpy().astype(np.uint64)
assert np.array_equal(c, oracle.partition_counts(4, 20001))
assert v.single_check(98) == 19 and v.single_check(10**6) == 17
v.close()
# K-LARGE (sieving primes above 2^21): a window at 1e13
v = Verifier(hi_max=10**13 + 1, p_max=65521, origin=10**13 - 2**21)
got, d = v.run(10**13 - 2**20, 10**13 + 1, dump=True)
want, wd = oracle.verify(10**13 - 2**20, 10**13 + 1, p_fast=65521, dump=True)
assert np.array_equal(d.cpu().numpy().astype(np.uint32), wd)
check(got, want, "1e13")
w_lo = (10**13 - 3) // 128 - 100
w = v.sieve_segment(w_lo, 100).cpu().numpy().view(np.uint64)
ob = oracle.sieve_window(3 + 128 * w_lo, 3 + 128 * (w_lo + 100))
assert np.array_equal(w, np.packbits(ob, bitorder="little").view(np.uint64))
x = torch.tensor([3215031751, 2**61 - 1, 561, 97], dtype=torch.int64)
assert v.is_prime(x).cpu().tolist() == [0, 1, 0, 1]
v.close()
torch.cuda.synchronize()
print("sanitize driver: all parity checks passed")
