"""NEXT-1: the paper's per-n gpu3 Phase-1 kernel
(three-way oracle) behind gb_verify_range_pern.  Bit-exact against
the CPU oracle and, field by field and n by n, against the product path (the
inverted bulk marking of gb_verify_range)."""
import numpy as np
import pytest

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


def same(got, want, what):
    for k in oracle.AGG_FIELDS:
        assert got[k] == want[k], (what, k, got[k], want[k])
    assert np.array_equal(np.asarray(got["hist"], dtype=np.int64), np.asarray(want["hist"], dtype=np.int64)), what


def test_pern_C1_1e6_vs_oracle(V):
    got, d = V.run(4, 10**6 + 1, dump=True, mode="pern")
    want, wd = oracle.verify(4, 10**6 + 1, p_fast=65521, dump=True)
    assert np.array_equal(d.cpu().numpy().astype(np.uint32), wd)
    same(got, want, "1e6")


@pytest.mark.parametrize("center", [10**9, 10**11, 10**12])
def test_pern_equals_bulk(V, center):
    rng = np.random.default_rng(SEED + center % 1000003)
    lo = int(rng.integers(center // 2, center - 2**24)) & ~1
    hi = lo + 2**24 + int(rng.integers(0, 300))                  # ragged tail
    for a, b in ((lo, hi), (center - 2**22, center + 1)):
        gb_, db = V.run(a, b, dump=True)
        gp, dp = V.run(a, b, dump=True, mode="pern")
        assert torch.equal(db, dp), (a, b)
        same(gp, gb_, (a, b))


@pytest.mark.parametrize("p_max", [5, 97])
def test_pern_forced_fallback(V, p_max):
    got, d = V.run(4, 10**5 + 1, p_max=p_max, dump=True, mode="pern")
    want, wd = oracle.verify(4, 10**5 + 1, p_fast=p_max, dump=True)
    assert got["fastpath_unresolved"] > 0
    assert np.array_equal(d.cpu().numpy().astype(np.uint32), wd)
    same(got, want, p_max)


def test_pern_segment_boundaries(V):
    """A range over several 2^28-even per-n segments (and the MR64 branch for q
    below each segment start) equals the bulk path n by n."""
    lo, hi = 10**12 - 2**29 - 2**20 - 1234, 10**12 + 1
    gb_, db = V.run(lo, hi, dump=True)
    gp, dp = V.run(lo, hi, dump=True, mode="pern")
    assert torch.equal(db, dp)
    same(gp, gb_, "segments")
