"""GPU parity in config C5's window [4e18 - 1e11, 4e18) (BASELINE.json configs[4];
SURVEY.md section 8(d) C5): base primes to isqrt(4e18 - 1) = 1,999,999,999, the
K-LARGE L2 mask for sieving primes above the carried range, 64-bit offsets.

Pins independent of the oracle: pi(2e9) (published), the two-method window prime
counts and the MR-computed golden points of SURVEY.md Appendix A.  Oracle parity:
aggregates, histogram and the SHA-256 of every per-n dump of the windows in
tests/golden/verify_4e18_windows.json (scripts/make_golden_4e18.py, oracle only).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, read_pairs
from oracle import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOP = 4 * 10**18
BOT = TOP - 10**11
CHK_DEF = "chk = sum n*p_min(n)"   # goldens written since round 2 (scripts/make_golden*.py)


@pytest.fixture(scope="module")
def V():
    from paper_2603_02621_b200.verifier import Verifier
    v = Verifier(hi_max=TOP, p_max=65521, origin=BOT)
    yield v
    v.close()


def test_base_table_to_2e9(V):
    # pi(2e9) = 98,222,287 (published), minus the prime 2
    assert V.R == 1999999999
    assert V.n_base == 98222287 - 1


@pytest.mark.parametrize("a,b,count", [(TOP - 10**6, TOP, 23281), (BOT, BOT + 10**6, 23249)])
def test_sieve_window_counts(V, a, b, count):
    """primes in [a, b), agreeing between a byte sieve and 12-base MR.
    The context sieves words whose every odd q has isqrt(q) <= R = isqrt(4e18 - 1):
    the word holding 4e18 + 1 is out of its range (GB_ERANGE), so the top few odd q
    of the first window are tested by the device MR64 instead."""
    from paper_2603_02621_b200 import gb
    w_lo = ((a - 3) // 2) // 64
    w_hi = min(((b - 1 - 3) // 2) // 64 + 1, (TOP - 3) // 128)
    with pytest.raises(gb.GBError):
        V.sieve_segment((TOP - 3) // 128, 1)
    w = V.sieve_segment(w_lo, w_hi - w_lo).cpu().numpy().view(np.uint64)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little").astype(bool)
    q = np.uint64(3 + 128 * w_lo) + np.uint64(2) * np.arange(bits.size, dtype=np.uint64)
    sel = (q >= np.uint64(a)) & (q < np.uint64(b))
    n = int(bits[sel].sum())
    q_top = 3 + 128 * w_hi                          # first odd q not covered by the words
    if q_top < b:
        rest = torch.arange(q_top, b, 2, dtype=torch.int64)
        n += int(V.is_prime(rest).sum())
    assert n == count


def test_sieve_segment_vs_oracle_4e18(V):
    """K-SIEVE word for word against the oracle's byte sieve at the top of the C5
    window (base primes up to 2e9: the K-LARGE mask path of gb_sieve_segment)."""
    w_lo = (TOP - 3) // 128 - 4096
    got = V.sieve_segment(w_lo, 4096).cpu().numpy().view(np.uint64)
    a = 3 + 128 * w_lo
    ob = oracle.sieve_window(a, a + 128 * 4096)
    bits = np.packbits(ob, bitorder="little").view(np.uint64)
    assert np.array_equal(got, bits)


def test_golden_points(V):
    for n, p in read_pairs("pmin_points_4e18.txt"):
        got, d = V.run(n, n + 1, dump=True)
        assert int(d.cpu()[0]) == p, n
        assert got["max_pmin"] == p and got["max_pmin_n"] == n


def _golden():
    path = os.path.join(GOLDEN, "verify_4e18_windows.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/verify_4e18_windows.json not generated yet")
    return json.load(open(path))


def test_windows_vs_oracle_golden(V):
    doc = _golden()
    for w in doc["windows"]:
        got, d = V.run(w["lo"], w["hi"], dump=True)
        g = w["result"]
        for k in oracle.AGG_FIELDS:
            assert got[k] == g[k], (w["lo"], k, got[k], g[k])
        hist = np.zeros(oracle.NBINS, np.int64)
        for i, c in g["hist"].items():
            hist[int(i)] = c
        assert np.array_equal(np.asarray(got["hist"]), hist), w["lo"]
        dd = d.cpu().numpy().astype("<u4")
        assert hashlib.sha256(dd.tobytes()).hexdigest() == w["dump_sha256"], w["lo"]
        ns = np.uint64(w["lo"] + (w["lo"] & 1)) + np.uint64(2) * np.arange(dd.size, dtype=np.uint64)
        if doc["chk_def"].startswith(CHK_DEF):
            assert int((ns * dd.astype(np.uint64)).sum()) & ((1 << 64) - 1) == g["chk"]


def test_pern_mode_golden_window(V):
    """NEXT-1 per-n kernel (three-way oracle: small bitset / segment bitset / MR64)
    on the top golden window: same aggregates and per-n dump hash."""
    w = _golden()["windows"][0]
    got, d = V.run(w["lo"], w["hi"], dump=True, mode="pern")
    for k in oracle.AGG_FIELDS:
        assert got[k] == w["result"][k], k
    assert hashlib.sha256(d.cpu().numpy().astype("<u4").tobytes()).hexdigest() == w["dump_sha256"]


def test_chunk_boundaries_and_composition(V):
    """A range spanning several K-LARGE chunks equals the sum of pieces whose chunk
    boundaries fall elsewhere, aggregate by aggregate and n by n (P13)."""
    span = 2 * 2_100_000_000                      # > 2 chunks of 148 x 3 tiles (1.97M evens each)
    lo = BOT + 10**9
    whole, dw = V.run(lo, lo + span, dump=True)
    cuts = [lo, lo + 777_777_778, lo + 2_500_000_002, lo + span]
    r = V.new_result()
    parts = []
    for a, b in zip(cuts, cuts[1:]):
        d = torch.zeros((b - a) // 2, dtype=torch.int32, device=V.device)
        V.verify(a, b, r, dump=d)
        parts.append(d)
    V.finalize(r)
    got = V.decode(r)
    for k in oracle.AGG_FIELDS:
        assert got[k] == whole[k], k
    assert got["hist"] == whole["hist"]
    assert torch.equal(torch.cat(parts), dw)
    assert whole["verified"] == whole["evens"] == span // 2 and whole["unresolved"] == 0


def test_full_c5_window_vs_oracle_golden(V):
    """Config C5 in full: every even n in [4e18 - 1e11, 4e18) (5e10 evens), all
    aggregates and the histogram vs the oracle's golden (scripts/make_golden.py
    --window c5; 1,572 s on 8 host cores)."""
    import json as _json
    path = os.path.join(GOLDEN, "verify_c5_4e18.json")
    doc = _json.load(open(path))
    got, _ = V.run(BOT, TOP)
    g = doc["result"]
    for k in oracle.AGG_FIELDS:
        assert got[k] == g[k], (k, got[k], g[k])
    hist = np.zeros(oracle.NBINS, np.int64)
    for i, c in g["hist"].items():
        hist[int(i)] = c
    assert np.array_equal(np.asarray(got["hist"]), hist)
