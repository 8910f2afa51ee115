"""GPU parity: libgb (C-ABI, sm_100a kernels) vs the CPU oracle, element by
element on the same inputs.  Integer path, so the bar is bit-exact everywhere:
every bitset word, every minimal p, every aggregate and histogram bin.

Inputs are number-theoretic ranges (deterministic; no value distribution to
choose).  Sampled windows use a seeded numpy generator (seed 20260302).
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, read_pairs
from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
SEED = 20260302
U64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def V():
    from paper_2603_02621_b200.verifier import Verifier
    v = Verifier(hi_max=10**12 + 1, p_max=65521)
    yield v
    v.close()


@pytest.fixture(scope="module")
def V1e6():
    """the paper's P_SMALL = 10^6 fast-path bound"""
    from paper_2603_02621_b200.verifier import Verifier
    v = Verifier(hi_max=10**12 + 1, p_max=10**6)
    yield v
    v.close()


def pack_odd_bytes(b):
    """oracle bytes (one per odd) -> paper's u64 word layout, independent of libgb"""
    n = len(b)
    pad = (-n) % 64
    bits = np.packbits(np.concatenate([b, np.zeros(pad, np.uint8)]), bitorder="little")
    return bits.view(np.uint64)


def assert_same(got, want, what=""):
    for k in oracle.AGG_FIELDS:
        assert got[k] == want[k], (what, k, got[k], want[k])
    assert np.array_equal(np.asarray(got["hist"], dtype=np.int64), want["hist"]), (what, "hist")


def run_both(V, lo, hi, p_max=65521, cap=None, dump=True):
    got, d = V.run(lo, hi, p_max=p_max, dump=dump, cap=cap)
    want, wd = oracle.verify(lo, hi, p_fast=p_max, cap=U64 if cap is None else cap, dump=dump)
    return got, (d.cpu().numpy().astype(np.uint32) if d is not None else None), want, wd


# ---------------------------------------------------------------- K-BASE
def test_kbase_resident_table(V):
    """K-BASE: the resident odd bitset of [3, R] and the u32 list, read straight
    out of the caller-owned workspace tensor, vs the oracle's sieve."""
    from paper_2603_02621_b200 import gb
    n_base, R = V.n_base, V.R
    assert R == 10**6
    assert n_base == 78498 - 1                     # pi(1e6) = 78,498, minus p = 2
    d_bits, d_primes = gb.gb_ctx_tables(V.ctx)
    base = V.workspace.data_ptr()
    nw = ((R - 3) // 2) // 64 + 1
    ws = V.workspace.cpu().numpy()
    bits = ws[d_bits - base: d_bits - base + 8 * nw].view(np.uint64)
    primes = ws[d_primes - base: d_primes - base + 4 * n_base].view(np.uint32)
    ob = oracle.sieve_window(3, R + 1)
    assert np.array_equal(bits, pack_odd_bytes(ob))
    assert np.array_equal(primes, 3 + 2 * np.flatnonzero(ob).astype(np.uint32))


# ---------------------------------------------------------------- K-SIEVE
@pytest.mark.parametrize("word_lo,n_words", [
    (0, 1), (0, 7813), (3, 20000), (0, 65536 + 17),
    ((10**9 - 2**24 - 3) // 128, 2**24 // 128 + 5),
    ((10**12 - 2**24 - 3) // 128, 2**24 // 128),
    ((10**12 - 3) // 128 - 100000, 99999),
    (1, 1), (2, 1), (30719, 3), (30720 * 3 - 7, 30720 + 11),     # one-word and tile-straddling windows
    ((10**11) // 128 + 5, 3 * 30720 * 148 + 1001),              # more tiles than CTAs (carried offsets)
])
def test_sieve_segment_parity(V, word_lo, n_words):
    got = V.sieve_segment(word_lo, n_words).cpu().numpy().view(np.uint64)
    a = 3 + 128 * word_lo
    b = a + 128 * n_words
    want = pack_odd_bytes(oracle.sieve_window(a, b))
    assert np.array_equal(got, want)


def test_sieve_popcount_pi_1e9(V):
    # popcount over odd q in [3, 1e9] + 1 (the prime 2) = pi(1e9) = 50,847,534 (BASELINE.json pin)
    nw = (10**9 - 3) // 128 + 1
    w = V.sieve_segment(0, nw)
    top = (10**9 - 3) // 2 + 1                   # odd q <= 1e9 are bits [0, top)
    arr = w.cpu().numpy().view(np.uint64)
    full = int(np.unpackbits(arr[: top // 64].view(np.uint8)).sum())
    last = int(arr[top // 64]) & ((1 << (top % 64)) - 1)
    assert full + bin(last).count("1") + 1 == 50847534


def test_sieve_errors(V):
    from paper_2603_02621_b200 import gb
    out = torch.empty(4, dtype=torch.int64, device=V.device)
    with pytest.raises(gb.GBError) as e:
        gb.gb_sieve_segment(V.ctx, (10**13) // 128, 4, out, V.stream)   # needs primes > 1e6
    assert e.value.status == gb.GB_ERANGE


# ---------------------------------------------------------------- verify
def test_verify_C1_1e6_dump(V):
    got, d, want, wd = run_both(V, 4, 10**6 + 1)
    assert np.array_equal(d, wd)
    assert_same(got, want, "C1")
    assert got["evens"] == 499999 and got["max_pmin"] == 523 and got["max_pmin_n"] == 503222


def test_verify_golden_4_200(V):
    got, d = V.run(4, 201, dump=True)
    gold = read_pairs("pmin_4_200.txt", sep=":")
    assert [(4 + 2 * i, int(p)) for i, p in enumerate(d.cpu().numpy())] == gold


def test_verify_points_large_n(V):
    for n, p in read_pairs("pmin_points.txt"):
        got, d = V.run(n, n + 1, dump=True)
        assert got["evens"] == 1 and int(d.cpu()[0]) == p, n


EDGE = [(4, 5), (4, 6), (4, 7), (5, 6), (5, 7), (6, 7), (7, 9), (130, 131), (131, 133), (0, 4),
        (10, 10), (4, 130), (4, 131), (4, 132), (4, 133), (62, 67), (64, 200), (100, 4200),
        (4, 65536 * 2 + 1), (1048576 - 6, 1048576 + 7), (2**21 + 2, 2**21 + 2 + 2 * 524288 + 66),
        (10**6 - 1, 10**6 + 1)]


@pytest.mark.parametrize("lo,hi", EDGE)
def test_verify_edges(V, lo, hi):
    got, d, want, wd = run_both(V, lo, hi)
    if wd is not None and len(wd):
        assert np.array_equal(d, wd)
    assert_same(got, want, (lo, hi))


@pytest.mark.parametrize("p_max", [3, 5, 7, 97, 1009, 65521])
def test_pmax_invariance_and_forced_fallback(V, p_max):
    # SPEC.md:345 / SURVEY P11: every field but fastpath_unresolved is p_max-invariant
    got, d, want, wd = run_both(V, 4, 10**5 + 1, p_max=p_max)
    assert np.array_equal(d, wd)
    assert_same(got, want, p_max)
    if p_max <= 7:
        assert got["fastpath_unresolved"] > 0 and got["unresolved"] == 0


def test_fallback_cap_counterexample_path(V):
    # test hook: with p_max = 5 and the fallback capped at 7, every n with
    # p_min > 7 is reported unresolved (a reproducible "counterexample")
    full, fd = oracle.verify(4, 10**5 + 1, dump=True)
    got, d = V.run(4, 10**5 + 1, p_max=5, dump=True, cap=7)
    d = d.cpu().numpy().astype(np.uint32)
    assert np.array_equal(d, np.where(fd > 7, 0, fd))
    assert got["unresolved"] == int((fd > 7).sum()) and got["first_unresolved_n"] == 98
    assert got["hist"][0] == got["unresolved"]


def test_paper_psmall_1e6(V1e6):
    # the paper's P_SMALL = 10^6: halo of 15,626 words
    got, d, want, wd = run_both(V1e6, 4, 3 * 10**6 + 1, p_max=10**6)
    assert np.array_equal(d, wd)
    assert_same(got, want, "psmall")
    lo = 10**12 - 2**22
    got, d, want, wd = run_both(V1e6, lo, 10**12 + 1, p_max=10**6)
    assert np.array_equal(d, wd)
    assert_same(got, want, "psmall-top")


def test_verify_1e9_aggregates(V):
    g = json.load(open(os.path.join(GOLDEN, "verify_1e09.json")))["result"]
    got, _ = V.run(4, 10**9 + 1, dump=False)
    for k in oracle.AGG_FIELDS:
        assert got[k] == g[k], k
    hist = np.zeros(oracle.NBINS, np.int64)
    for i, c in g["hist"].items():
        hist[int(i)] = c
    assert np.array_equal(np.asarray(got["hist"]), hist)


@pytest.mark.parametrize("center", [10**9, 10**11, 10**12])
def test_sampled_windows_dump(V, center):
    rng = np.random.default_rng(SEED + center % 1000003)
    for _ in range(2):
        lo = int(rng.integers(center // 2, center - 2**23)) & ~1
        hi = lo + 2**23 + int(rng.integers(0, 300))
        got, d, want, wd = run_both(V, lo, hi)
        assert np.array_equal(d, wd), (lo, hi)
        assert_same(got, want, (lo, hi))
    # the very top of [4, N]
    got, d, want, wd = run_both(V, center - 2**22, center + 1)
    assert np.array_equal(d, wd)
    assert_same(got, want, "top")


def test_shard_invariance_virtual_ranks(V):
    # the same result for R in {1,2,4,8} strips round-robin (virtual ranks
    # executed one after another on one GPU, reduced on the device by accumulation)
    from paper_2603_02621_b200 import dist
    lo, hi = 4, 2 * 10**8 + 1
    ref, _ = V.run(lo, hi)
    for world in (2, 4, 8):
        r = V.new_result()
        for rank in range(world):
            for a, b in dist.rank_strips(dist.plan_strips(lo, hi, 32 * world), rank, world):
                V.verify(a, b, r)
        V.finalize(r)
        got = V.decode(r)
        for k in oracle.AGG_FIELDS:
            assert got[k] == ref[k], (world, k)
        assert got["hist"] == ref["hist"]


@pytest.mark.parametrize("N,name", [("1e10", "verify_1e10"), ("1e11", "verify_1e11"), ("1e12", "verify_1e12")])
def test_golden_aggregates(V, N, name):
    """Aggregates over [4, N] vs golden JSONs written by the oracle (scripts/make_golden.py).
    (Per-n parity over the same ranges: test_gpu_fullscale.py.)"""
    path = os.path.join(GOLDEN, f"{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    doc = json.load(open(path))
    g = doc["result"]
    got, _ = V.run(4, int(float(N)) + 1, dump=False)
    for k in oracle.AGG_FIELDS:
        assert got[k] == g[k], k
    hist = np.zeros(oracle.NBINS, np.int64)
    for i, c in g["hist"].items():
        hist[int(i)] = c
    assert np.array_equal(np.asarray(got["hist"]), hist)


# ---------------------------------------------------------------- MR64
def test_mr64_vectors(V):
    vals = {3215031751: 0, 3825123056546413051: 0, 2**61 - 1: 1, 561: 0, 41041: 0, 825265: 0,
            1: 0, 0: 0, 2: 1, 3: 1, 4: 0, 37: 1, 41: 1, 1681: 0, 999999999989: 1,
            18446744073709551557: 1, 18446744073709551615: 0, 4294967291: 1, 4294967297: 0}
    xs = list(vals)
    t = torch.tensor([x - (1 << 64) if x >= 1 << 63 else x for x in xs], dtype=torch.int64)
    got = V.is_prime(t).cpu().tolist()
    assert got == [vals[x] for x in xs]


def test_mr64_exhaustive_below_1e6(V):
    # SPEC.md:165 exhaustive equivalence with trial division for n < 1e6 (oracle window sieve
    # is trial-division-equivalent, pinned in test_oracle.py)
    x = torch.arange(0, 10**6, dtype=torch.int64)
    got = V.is_prime(x).cpu().numpy()
    odd = oracle.sieve_window(3, 10**6)
    want = np.zeros(10**6, np.uint8)
    want[3::2] = odd
    want[2] = 1
    assert np.array_equal(got, want)
    # and a seeded sample of large odd n against trial division in the oracle
    rng = np.random.default_rng(SEED)
    xs = [int(v) | 1 for v in rng.integers(10**12, 10**13, size=300)]
    got = V.is_prime(torch.tensor(xs, dtype=torch.int64)).cpu().tolist()
    assert got == [int(oracle.is_prime_td(v)) for v in xs]


def test_verify_errors(V):
    from paper_2603_02621_b200 import gb
    r = V.new_result()
    for args, st in [((10, 4, 65521), gb.GB_EINVAL), ((4, 100, 2), gb.GB_EINVAL),
                     ((4, 100, 70000), gb.GB_EINVAL), ((4, 10**12 + 3, 65521), gb.GB_ERANGE)]:
        with pytest.raises(gb.GBError) as e:
            gb.gb_verify_range(V.ctx, *args, r, None, V.stream)
        assert e.value.status == st, args
