"""Pins for the CPU oracle (oracle/gb_oracle.c) against values the paper and the
mathematics fix -- never against the oracle itself.  CPU only (-m "not gpu").

Each pin is chosen so a plausible oracle bug fails it:
  * sieve:   published pi(x) (drops / extra clears), window counts at 1e12
             (base-prime bound, start offsets), trial division on windows;
  * scan:    brute force by trial division for n <= 20000 (wrong order / bound),
             golden n = 4..200 and large-n points (window below segment),
             record table A025018 (tie-break to the smallest n),
             closed forms hist[3] = pi(N-3) - 1 and hist[5] = pi(N-5) - 1 - pi2
             (wrong bin / dropped term), printed evens = N/2 - 1 (range ends);
  * aggregation: additivity over disjoint ranges, cap / p_fast semantics.
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, read_pairs
from oracle import oracle

U64 = (1 << 64) - 1


def td_prime(x):
    """Independent Python trial division (test-local)."""
    if x < 2:
        return False
    if x % 2 == 0:
        return x == 2
    d = 3
    while d * d <= x:
        if x % d == 0:
            return False
        d += 2
    return True


def brute_pmin(n):
    """p_min by the definition, trial division of both p and q."""
    for p in range(2, n // 2 + 1):
        if td_prime(p) and td_prime(n - p):
            return p
    return 0


def prime_index_bins(limit=65521):
    """1-based index of each prime <= limit (bin numbering R5)."""
    idx, k = {}, 0
    for x in range(2, limit + 1):
        if td_prime(x):
            k += 1
            idx[x] = k
    return idx


PUB = json.load(open(os.path.join(GOLDEN, "pi_published.json")))
AGG = json.load(open(os.path.join(GOLDEN, "aggregates.json")))


def test_isqrt_exact():
    assert oracle.isqrt(4 * 10**18 - 1) == 1999999999
    assert oracle.isqrt(U64) == 2**32 - 1
    for r in (1, 2, 3, 1000, 10**6, 2**31 - 1, 2**32 - 1, 1999999999):
        assert oracle.isqrt(r * r) == r
        assert oracle.isqrt(r * r - 1) == r - 1
        assert oracle.isqrt(r * r + 2 * r) == r


def test_trial_division_examples():
    # SPEC.md:161 strong pseudoprime 3,215,031,751 = 151*751*28351 is composite
    assert not oracle.is_prime_td(3215031751)
    assert oracle.is_prime_td(2**31 - 1)
    assert oracle.is_prime_td(999999999989)          # largest prime < 1e12
    for c in (561, 41041, 825265, 1, 0, 4, 91):        # Carmichael numbers, units, 91 = 7*13
        assert not oracle.is_prime_td(c)
    for x in range(0, 3000):
        assert oracle.is_prime_td(x) == td_prime(x)


@pytest.mark.parametrize("x", ["1000", "1000000", "10000000", "100000000", "1000000000"])
def test_prime_pi_published(x):
    assert oracle.prime_pi(int(x)) == PUB["pi"][x]


def test_prime_pi_small_exhaustive():
    primes = [x for x in range(2, 5000) if td_prime(x)]
    for x in (2, 3, 4, 10, 97, 100, 101, 4999):
        assert oracle.prime_pi(x) == sum(1 for p in primes if p <= x)


def test_sieve_window_vs_trial_division():
    # [1e8+1, 1e8+1e4] matches trial division; 999,983 prime.
    for a, b in ((3, 10001), (10**8 + 1, 10**8 + 10**4 + 1), (999001, 1000001), (4294967291, 4294977291)):
        got = oracle.sieve_window(a, b)
        want = np.array([td_prime(q) for q in range(a, b, 2)], dtype=np.uint8)
        assert np.array_equal(got, want), (a, b)
    w = oracle.sieve_window(999001, 1000001)
    assert w[(999983 - 999001) // 2] == 1


def test_window_count_at_1e12():
    # primes in [1e12 - 1e6, 1e12) = 36,400 (two methods)
    w = oracle.sieve_window(10**12 - 10**6 + 1, 10**12)
    assert int(w.sum()) == PUB["window_prime_counts"]["[999999000000,1000000000000)"]


def test_brute_force_small():
    # every even n <= 20000 against the definition (trial division of p and q)
    hi = 20001
    r, d = oracle.verify(4, hi, dump=True, threads=2)
    want = np.array([brute_pmin(n) for n in range(4, hi, 2)], dtype=np.uint32)
    assert np.array_equal(d, want)
    assert r["evens"] == len(want) and r["unresolved"] == 0
    assert r["sum_pmin"] == int(want.sum())
    ns = np.arange(4, hi, 2, dtype=np.uint64)
    assert r["chk"] == int((want.astype(np.uint64) * ns).sum()) & U64
    idx = prime_index_bins()
    h = np.zeros(oracle.NBINS, dtype=np.int64)
    for p in want:
        h[idx[int(p)]] += 1
    assert np.array_equal(r["hist"], h)


def test_golden_4_200():
    gold = read_pairs("pmin_4_200.txt", sep=":")
    r, d = oracle.verify(4, 201, dump=True, threads=1)
    assert [(4 + 2 * i, int(p)) for i, p in enumerate(d)] == gold


def test_golden_points_large_n():
    for n, p in read_pairs("pmin_points.txt"):
        r, d = oracle.verify(n, n + 1, dump=True, threads=1)
        assert r["evens"] == 1 and int(d[0]) == p, n


def test_records_A025018_to_1e8():
    N = 10**8
    r, d = oracle.verify(4, N + 1, dump=True)
    run = np.maximum.accumulate(d)
    first = np.flatnonzero(np.concatenate(([True], run[1:] > run[:-1])))
    got = [(4 + 2 * int(i), int(d[i])) for i in first]
    want = [(n, p) for n, p in read_pairs("records_A025018.txt") if n <= N]
    assert got == want
    assert (r["max_pmin"], r["max_pmin_n"]) == want[-1][::-1]


@pytest.mark.parametrize("N", ["1000000", "100000000", "1000000000"])
def test_aggregates_appendix_A(N):
    n = int(N)
    r, _ = oracle.verify(4, n + 1)
    a = AGG[N]
    assert r["evens"] == a["evens"] == n // 2 - 1          # PAPER.md:213-216 "Even n checked"
    assert r["verified"] == r["evens"] and r["unresolved"] == 0
    assert r["sum_pmin"] == a["sum_pmin"]
    assert (r["max_pmin"], r["max_pmin_n"]) == (a["max_pmin"], a["max_pmin_n"])
    idx = prime_index_bins(100)
    for p, c in a["hist_by_p"].items():
        assert r["hist"][idx[int(p)]] == c, p
    if "distinct_pmin" in a:
        assert int((r["hist"][1:] > 0).sum()) == a["distinct_pmin"]
    assert int(r["hist"].sum()) == r["evens"]


@pytest.mark.parametrize("N", ["1000000", "100000000", "1000000000"])
def test_closed_form_bins(N):
    """hist[p=3] = pi(N-3) - 1 ; hist[p=5] = pi(N-5) - 1 - pi2(N).
    For these N no prime lies in (N-5, N], so pi(N-3) = pi(N-5) = pi(N)."""
    n = int(N)
    r, _ = oracle.verify(4, n + 1)
    pi, pi2 = PUB["pi"][N], PUB["pi2"][N]
    assert r["hist"][2] == pi - 1
    assert r["hist"][3] == pi - 1 - pi2


def test_sum_n_pmin_1e6():
    # SURVEY.md Appendix A (an independent brute-force program): sum n * p_min over
    # [4, 1e6] = 5,216,083,445,938 -- the oracle's chk (SURVEY 8(b) definition; no
    # wrap below 2^64 here), and the same from its dump
    r, d = oracle.verify(4, 10**6 + 1, dump=True)
    ns = np.arange(4, 10**6 + 1, 2, dtype=np.int64)
    assert int((ns * d.astype(np.int64)).sum()) == AGG["1000000"]["sum_n_pmin"]
    assert r["chk"] == AGG["1000000"]["sum_n_pmin"]


def test_chunk_checksums():
    """Per-chunk chk (the golden format of scripts/make_golden.py): each chunk's
    value is sum n * p_min over its evens (from the dump, numpy uint64 wrap), for a
    range with a ragged last chunk and an odd lo, and for chunks smaller than the
    oracle's segments."""
    for lo, hi, ce in ((4, 300001, 1 << 14), (1001, 2 * 10**6 + 7, 1 << 16), (10**12 - 10**6 + 1, 10**12, 1 << 17)):
        r, d = oracle.verify(lo, hi, dump=True, chunk_evens=ce)
        ns = oracle.lo_even(lo) + 2 * np.arange(d.size, dtype=np.uint64)
        prod = ns * d.astype(np.uint64)
        want = [int(prod[i:i + ce].sum()) & U64 for i in range(0, d.size, ce)]
        assert [int(x) for x in r["chunk_chk"]] == want
        assert sum(want) & U64 == r["chk"]


def test_additivity_and_edges():
    full, dfull = oracle.verify(4, 300001, dump=True)
    parts = [(4, 777), (777, 778), (778, 65536), (65536, 65537), (65537, 300001)]
    acc = None
    for lo, hi in parts:
        r, _ = oracle.verify(lo, hi, threads=3)
        if acc is None:
            acc = r
            continue
        for k in ("evens", "verified", "fastpath_unresolved", "unresolved", "sum_pmin"):
            acc[k] += r[k]
        acc["chk"] = (acc["chk"] + r["chk"]) & U64
        acc["hist"] = acc["hist"] + r["hist"]
        if (r["max_pmin"], -r["max_pmin_n"]) > (acc["max_pmin"], -acc["max_pmin_n"]):
            acc["max_pmin"], acc["max_pmin_n"] = r["max_pmin"], r["max_pmin_n"]
    for k in ("evens", "verified", "sum_pmin", "chk", "max_pmin", "max_pmin_n"):
        assert acc[k] == full[k], k
    assert np.array_equal(acc["hist"], full["hist"])
    # empty / degenerate ranges
    assert oracle.verify(10, 10)[0]["evens"] == 0
    assert oracle.verify(0, 4)[0]["evens"] == 0
    assert oracle.verify(0, 5)[0]["evens"] == 1            # only n = 4
    assert oracle.verify(5, 6)[0]["evens"] == 0
    assert oracle.verify(7, 9)[0]["evens"] == 1            # only n = 8


def test_cap_and_pfast_semantics():
    # forced fallback: with p_fast = 5, every n with p_min > 5 is
    # a Phase-2 invocation; with cap = 5 those n become unresolved.
    r_full, d = oracle.verify(4, 100001, dump=True)
    r5, _ = oracle.verify(4, 100001, p_fast=5)
    assert r5["fastpath_unresolved"] == int((d > 5).sum()) > 0
    assert r5["unresolved"] == 0
    rc, dc = oracle.verify(4, 100001, cap=5, dump=True)
    assert rc["unresolved"] == int((d > 5).sum())
    assert np.array_equal(dc, np.where(d > 5, 0, d))
    first = 4 + 2 * int(np.flatnonzero(d > 5)[0])
    assert rc["first_unresolved_n"] == first == 30          # p_min(30) = 7
    assert rc["hist"][0] == rc["unresolved"]


@pytest.mark.parametrize("N,tag", [("1000000000", "1e09"), ("10000000000", "1e10"),
                                   ("100000000000", "1e11")])
def test_golden_files_match_appendix(N, tag):
    """The oracle-written golden JSONs agree with SURVEY Appendix A (computed by an
    independent throwaway program) and with published pi / pi2."""
    path = os.path.join(GOLDEN, f"verify_{tag}.json")
    if not os.path.exists(path):
        pytest.skip("golden not generated")
    g = json.load(open(path))["result"]
    a = AGG[N]
    assert g["evens"] == a["evens"] and g["sum_pmin"] == a["sum_pmin"]
    assert (g["max_pmin"], g["max_pmin_n"]) == (a["max_pmin"], a["max_pmin_n"])
    idx = prime_index_bins(100)
    for p, c in a["hist_by_p"].items():
        assert g["hist"][str(idx[int(p)])] == c
    assert g["hist"]["2"] == PUB["pi"][N] - 1
    assert g["hist"]["3"] == PUB["pi"][N] - 1 - PUB["pi2"][N]


def test_golden_1e12_closed_forms():
    """1e12 golden (oracle only) vs published pi(1e12), pi2(1e12)."""
    g = json.load(open(os.path.join(GOLDEN, "verify_1e12.json")))["result"]
    assert g["evens"] == 10**12 // 2 - 1
    assert g["hist"]["2"] == PUB["pi"]["1000000000000"] - 1 == 37607912017
    assert g["hist"]["3"] == PUB["pi"]["1000000000000"] - 1 - PUB["pi2"]["1000000000000"] == 35737326797
    assert g["unresolved"] == 0 and g["fastpath_unresolved"] == 0


def test_golden_4e18_windows_match_appendix():
    """The oracle-written C5 window goldens agree with SURVEY.md Appendix A's
    independent (12-base MR, no sieve) window maxima: 3,191 @ 3,999,999,999,998,238,538
    at the top of [4e18 - 1e11, 4e18) and 3,167 @ 3,999,999,900,003,045,538 at its
    bottom; every window is fully verified with no fallback."""
    path = os.path.join(GOLDEN, "verify_4e18_windows.json")
    doc = json.load(open(path))
    w = {(x["lo"], x["hi"]): x["result"] for x in doc["windows"]}
    top = w[(4 * 10**18 - 2**23, 4 * 10**18)]
    bot = w[(4 * 10**18 - 10**11, 4 * 10**18 - 10**11 + 2**23)]
    assert (top["max_pmin"], top["max_pmin_n"]) == (3191, 3999999999998238538)
    assert (bot["max_pmin"], bot["max_pmin_n"]) == (3167, 3999999900003045538)
    for r in w.values():
        assert r["evens"] == r["verified"] and r["fastpath_unresolved"] == 0 and r["unresolved"] == 0
        assert sum(r["hist"].values()) == r["evens"]


def test_golden_c5_window_consistency():
    """The full C5 golden (oracle only): 5e10 evens, all verified on the fast path,
    histogram sums to the evens, p_min below the known bound 9,781 for n <= 4e18
    (SURVEY P9), and its maximum is at least the top window's 3,191 (Appendix A)."""
    g = json.load(open(os.path.join(GOLDEN, "verify_c5_4e18.json")))["result"]
    assert g["evens"] == g["verified"] == 5 * 10**10
    assert g["fastpath_unresolved"] == 0 and g["unresolved"] == 0
    assert sum(g["hist"].values()) == g["evens"]
    assert 3191 <= g["max_pmin"] <= 9781
    assert 4 * 10**18 - 10**11 <= g["max_pmin_n"] < 4 * 10**18


@pytest.mark.parametrize("tag", ["1e06", "1e09", "1e10", "1e11", "1e12", "c5_4e18"])
def test_golden_chunk_files_consistent(tag):
    """Every per-chunk checksum file (oracle-written) has one entry per 2^24 evens of
    its range and sums, mod 2^64, to the golden's sum n * p_min."""
    doc = json.load(open(os.path.join(GOLDEN, f"verify_{tag}.json")))
    chk = np.load(os.path.join(GOLDEN, doc["chunk_chk_file"]))
    evens = doc["result"]["evens"]
    assert chk.dtype == np.uint64 and chk.size == -(-evens // doc["chunk_evens"])
    assert int(chk.sum(dtype=np.uint64)) == doc["result"]["chk"]


# ---------------------------------------------------------------- c(n) (NEXT-4)
def test_partition_counts_hand_values():
    """c(n) = #{p prime <= n/2 : n - p prime} (R13): 4 = 2+2; 10 = 3+7 = 5+5;
    100 = 3+97 = 11+89 = 17+83 = 29+71 = 41+59 = 47+53."""
    c = oracle.partition_counts(4, 101)
    want = {4: 1, 6: 1, 8: 1, 10: 2, 12: 1, 14: 2, 16: 2, 18: 2, 20: 2, 22: 3, 100: 6}
    for n, v in want.items():
        assert int(c[(n - 4) // 2]) == v, n


def test_partition_counts_vs_convolution():
    """r(n) = number of ORDERED prime pairs (p, q), p + q = n, is the self-convolution of
    the prime indicator (numpy's convolve: a library routine, not the oracle's loop);
    c(n) = (r(n) + [n/2 prime]) / 2."""
    N = 40000
    P = np.zeros(N + 1, dtype=np.int64)
    for x in range(2, N + 1):
        P[x] = td_prime(x)
    r = np.convolve(P, P)[: N + 1]
    c = oracle.partition_counts(4, N + 1)
    n = np.arange(4, N + 1, 2)
    want = (r[n] + P[n // 2]) // 2
    assert np.array_equal(c.astype(np.int64), want)


def test_partition_counts_sum_identity():
    """sum of c(n) over even n <= N counts the unordered prime pairs p <= q with
    p + q <= N and p + q even: 1 (2 + 2) + sum over odd primes p <= N/2 of
    #{odd primes q : p <= q <= N - p} -- prefix counts of a test-local sieve; also
    an odd lo and a window at 1e7."""
    N = 10**6
    s = np.ones(N + 1, dtype=bool)
    s[:2] = False
    for i in range(2, 1001):
        if s[i]:
            s[i * i::i] = False
    odd = s.copy()
    odd[2] = False
    pref = np.cumsum(odd)
    ps = np.flatnonzero(odd[: N // 2 + 1])
    want = 1 + int((pref[N - ps] - pref[ps - 1]).sum())
    c = oracle.partition_counts(4, N + 1)
    assert int(c.sum()) == want
    assert int(c[-1]) == 5402                       # c(10^6), the window end
    w = oracle.partition_counts(10**6 - 999, 10**6 + 1)
    assert np.array_equal(w, c[-500:])
