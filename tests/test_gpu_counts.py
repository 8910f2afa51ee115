"""NEXT-4 on the GPU: Goldbach partition counts c(n) (gb_partition_counts, the
popcount-AND of the odd prime bitset against its reversed shifts) vs the CPU
oracle's plain scan (oracle.partition_counts), element by element."""
import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def V():
    from paper_2603_02621_b200.verifier import Verifier
    v = Verifier(hi_max=10**9 + 2**20)
    yield v
    v.close()


def test_counts_full_1e6(V):
    got = V.partition_counts(4, 10**6 + 1).cpu().numpy().astype(np.uint64)
    want = oracle.partition_counts(4, 10**6 + 1)
    assert np.array_equal(got, want)
    assert int(got[0]) == 1 and int(got[(100 - 4) // 2]) == 6 and int(got[-1]) == 5402


@pytest.mark.parametrize("lo,hi", [(4, 5), (4, 7), (5, 6), (6, 7), (7, 100), (123, 4567), (1000, 1066),
                                   (2**16 - 2, 2**16 + 2 * 96 + 1), (999_000, 1_000_001), (30, 31)])
def test_counts_edges(V, lo, hi):
    got = V.partition_counts(lo, hi).cpu().numpy().astype(np.uint64)
    want = oracle.partition_counts(lo, hi)
    assert np.array_equal(got, want), (lo, hi)


def test_counts_window_1e9(V):
    """a window at 1e9 (about 7.8e6 i-words per n: many work items per tile)"""
    lo, hi = 10**9 - 2 * 300 - 1, 10**9 + 1
    bits = V.sieve_segment(0, (hi - 3 + 127) // 128)
    got = V.partition_counts(lo, hi, bits=bits).cpu().numpy().astype(np.uint64)
    want = oracle.partition_counts(lo, hi)
    assert np.array_equal(got, want)


def test_counts_errors(V):
    from paper_2603_02621_b200 import gb
    bits = V.sieve_segment(0, 100)
    out = torch.empty(64, dtype=torch.int64, device=V.device)
    with pytest.raises(gb.GBError) as e:                    # bitset too short for hi
        gb.gb_partition_counts(V.ctx, 4, 3 + 128 * 100 + 2, bits, 100, out, V.stream)
    assert e.value.status == gb.GB_EINVAL
    with pytest.raises(gb.GBError) as e:
        gb.gb_partition_counts(V.ctx, 10, 4, bits, 100, out, V.stream)
    assert e.value.status == gb.GB_EINVAL
