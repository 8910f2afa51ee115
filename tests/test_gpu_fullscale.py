"""Full-scale per-n parity: every minimal p of the configured ranges, not only
their aggregates (BASELINE.json north_star: "every count, every minimal p").

* [4, 2e9] in ONE gb_verify_range call (508 tiles over 148 persistent CTAs: every
  CTA carries its sieve offsets through >= 3 tiles) dumped and compared element by
  element with the oracle's dump of the same range.
* [4, 1e10], [4, 1e11], [4, 1e12] and the C5 window [4e18 - 1e11, 4e18): the GPU
  dump of the whole range (in calls of 2^30 evens through one device buffer) is
  reduced on the device to chk = sum n * p_min mod 2^64 per chunk of 2^24 evens,
  the checksum SURVEY.md 8(b) defines, and compared chunk by chunk with the
  oracle-written goldens (scripts/make_golden.py: tests/golden/chk_<tag>.npy);
  a p_min placed on the wrong n, or a wrong p_min anywhere, changes its chunk.
  The aggregates and the histogram are compared with the golden JSON as well.

The reduction is test code (torch on the device, exact int64 pieces recombined
mod 2^64 in Python): it is not the product path, and the goldens come from the
oracle only.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

U64 = (1 << 64) - 1
CHUNK = 1 << 24                 # evens per golden chunk (scripts/make_golden.py)
CALL_EVENS = 1 << 30            # evens per gb_verify_range call (4 GiB dump)


def chunk_checksums(V, lo, hi, p_max=65521, call_evens=CALL_EVENS):
    """GPU: per-chunk sum n * p_min mod 2^64 over [lo, hi) (lo even), plus the
    accumulated result vector of the same calls."""
    assert lo % 2 == 0 and call_evens % CHUNK == 0
    dev = V.device
    buf = torch.empty(call_evens, dtype=torch.int32, device=dev)
    ar = torch.arange(CHUNK, dtype=torch.int64, device=dev)
    r = V.new_result()
    out = []
    n0 = lo
    while n0 < hi:
        n1 = min(hi, n0 + 2 * call_evens)
        ne = (n1 - n0 + 1) // 2
        d = buf[:ne]
        V.verify(n0, n1, r, p_max=p_max, dump=d)
        nch = -(-ne // CHUNK)
        if nch * CHUNK != ne:
            buf[ne:nch * CHUNK].zero_()
        x = buf[:nch * CHUNK].view(nch, CHUNK).to(torch.int64)
        assert int(x.max()) < (1 << 14)          # keeps the int64 pieces below exact
        s0 = x.sum(dim=1)                        # sum p             < 2^38
        s1 = (x * ar).sum(dim=1)                 # sum i * p         < 2^62
        for c, (a, b) in enumerate(zip(s0.tolist(), s1.tolist())):
            base = n0 + 2 * CHUNK * c            # n of column i = base + 2 i
            out.append((base * a + 2 * b) & U64)
        n0 = n1
    V.finalize(r)
    return out, V.decode(r)


def load_golden(tag):
    path = os.path.join(GOLDEN, f"verify_{tag}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    doc = json.load(open(path))
    if "chunk_chk_file" not in doc:
        pytest.skip(f"{path} predates the per-chunk checksums")
    chk = np.load(os.path.join(GOLDEN, doc["chunk_chk_file"]))
    return doc, [int(x) for x in chk]


def compare_result(got, g):
    for k in oracle.AGG_FIELDS:
        assert got[k] == g[k], (k, got[k], g[k])
    hist = np.zeros(oracle.NBINS, np.int64)
    for i, c in g["hist"].items():
        hist[int(i)] = c
    assert np.array_equal(np.asarray(got["hist"]), hist)


def test_chunk_checksum_helper_matches_dump():
    """The device reduction is the plain definition: recompute it on the host with
    numpy uint64 (wrapping) from the same dump, on a range with a ragged chunk."""
    from paper_2603_02621_b200.verifier import Verifier
    v = Verifier(hi_max=10**8 + 1)
    lo, hi = 10**8 - 2 * CHUNK - 2 * 12345, 10**8 + 1
    got, _ = chunk_checksums(v, lo, hi, call_evens=CHUNK)
    _, d = oracle.verify(lo, hi, dump=True)
    ns = lo + 2 * np.arange(d.size, dtype=np.uint64)
    prod = ns * d.astype(np.uint64)
    want = [int(prod[i:i + CHUNK].sum()) & U64 for i in range(0, d.size, CHUNK)]
    assert got == want
    v.close()


def test_full_dump_4_2e9_one_call():
    """Every minimal p of [4, 2e9] from one call (>= 3 tiles per persistent CTA:
    the carried-offset path) equals the oracle's, n by n."""
    from paper_2603_02621_b200.verifier import Verifier
    N = 2 * 10**9
    v = Verifier(hi_max=N + 1)
    got, d = v.run(4, N + 1, dump=True)
    words = (N // 6) // 32 + 1
    assert -(-words // 20480) >= 3 * 148           # tiles per CTA >= 3
    want, wd = oracle.verify(4, N + 1, dump=True)
    dd = d.cpu().numpy().view(np.uint32)
    del d
    bad = np.flatnonzero(dd != wd)
    assert bad.size == 0, [(4 + 2 * int(i), int(dd[i]), int(wd[i])) for i in bad[:10]]
    for k in oracle.AGG_FIELDS:
        assert got[k] == want[k], k
    assert np.array_equal(np.asarray(got["hist"]), want["hist"])
    ns = 4 + 2 * np.arange(wd.size, dtype=np.uint64)
    assert int((ns * wd.astype(np.uint64)).sum()) & U64 == want["chk"]
    v.close()


@pytest.mark.parametrize("tag,lo,hi", [
    ("1e10", 4, 10**10 + 1),
    ("1e11", 4, 10**11 + 1),
    ("1e12", 4, 10**12 + 1),
    ("c5_4e18", 4 * 10**18 - 10**11, 4 * 10**18),
])
def test_per_chunk_checksums_vs_golden(tag, lo, hi):
    doc, want = load_golden(tag)
    assert (doc["lo"], doc["hi"], doc["chunk_evens"]) == (lo, hi, CHUNK)
    from paper_2603_02621_b200.verifier import Verifier
    v = Verifier(hi_max=hi, origin=lo if lo > 4 else 0)
    got, res = chunk_checksums(v, lo, hi)
    assert len(got) == len(want)
    bad = [i for i, (a, b) in enumerate(zip(got, want)) if a != b]
    assert not bad, f"{len(bad)} chunks differ, first at n = {lo + 2 * CHUNK * bad[0]}"
    compare_result(res, doc["result"])
    assert sum(got) & U64 == doc["result"]["chk"]
    v.close()
