"""NEXT-2 (the paper's gpu2 global resident bitset) and NEXT-3
(single_check) -- SURVEY.md section 8(f) -- against the oracle,
the golden files and the product path."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, read_pairs
from oracle import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def V():
    from paper_2603_02621_b200.verifier import Verifier
    v = Verifier(hi_max=10**9 + 1, p_max=65521)
    yield v
    v.close()


def test_resident_1e6_dump_vs_oracle(V):
    bits = V.sieve_segment(0, (10**6 + 1 - 3) // 128 + 1)
    got, d = V.run_resident(4, 10**6 + 1, bits, dump=True)
    want, wd = oracle.verify(4, 10**6 + 1, p_fast=65521, dump=True)
    assert np.array_equal(d.cpu().numpy().astype(np.uint32), wd)
    for k in oracle.AGG_FIELDS:
        assert got[k] == want[k], k


def test_resident_1e9_vs_golden(V):
    """gpu2 regime at N = 1e9: the whole 62.5 MB odd bitset of [3, 1e9] resident."""
    bits = V.sieve_segment(0, (10**9 + 1 - 3) // 128 + 1)
    got, _ = V.run_resident(4, 10**9 + 1, bits)
    g = json.load(open(os.path.join(GOLDEN, "verify_1e09.json")))["result"]
    for k in oracle.AGG_FIELDS:
        assert got[k] == g[k], k
    hist = np.zeros(oracle.NBINS, np.int64)
    for i, c in g["hist"].items():
        hist[int(i)] = c
    assert np.array_equal(np.asarray(got["hist"]), hist)


def test_resident_requires_covering_bitset(V):
    from paper_2603_02621_b200 import gb
    bits = V.sieve_segment(0, 100)
    with pytest.raises(gb.GBError) as e:
        V.run_resident(4, 3 + 128 * 100 + 2, bits)
    assert e.value.status == gb.GB_EINVAL


def test_single_check_golden_points(V):
    pts = read_pairs("pmin_4_200.txt", sep=":") + read_pairs("pmin_points.txt") + read_pairs("pmin_points_4e18.txt")
    for n, p in pts:
        assert V.single_check(n) == p, n


def test_single_check_vs_oracle_window(V):
    lo, hi = 10**12 - 20000, 10**12 + 1
    _, wd = oracle.verify(lo, hi, p_fast=65521, dump=True)
    rng = np.random.default_rng(20260302)
    for i in rng.choice(len(wd), 64, replace=False):
        n = lo + 2 * int(i)
        assert V.single_check(n) == int(wd[i]), n


def test_single_check_limits(V):
    from paper_2603_02621_b200 import gb
    assert V.single_check(4) == 2
    assert V.single_check(98) == 19
    assert V.single_check(98, p_limit=17) == 0           # no partition with p <= 17
    for bad in (3, 2, 99):
        with pytest.raises(gb.GBError):
            V.single_check(bad)
