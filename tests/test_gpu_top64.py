"""Edge of the accepted range: the window just below GB_HI_LIMIT = 2^62 (include/gb.h).
Base primes up to isqrt(2^62 - 1) = 2^31 - 1 (105 M), K-LARGE chunks, 64-bit offsets
-- against the CPU oracle n by n (the oracle first sieves its 2.1 GB byte table of
small primes on the host, so this test takes a minute or two)."""
import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HI = 2**62                          # GB_HI_LIMIT
LO = HI - 2**21


@pytest.fixture(scope="module")
def V():
    from paper_2603_02621_b200.verifier import Verifier
    v = Verifier(hi_max=HI, p_max=65521, origin=LO - 2**30)
    yield v
    v.close()


def test_top_of_u64_window_vs_oracle(V):
    assert V.R == oracle.isqrt(HI - 1) == 2**31 - 1
    from paper_2603_02621_b200 import gb
    assert gb.gb_ctx_workspace_bytes(HI + 2, 65521) == 0           # beyond GB_HI_LIMIT
    got, d = V.run(LO, HI, dump=True)
    want, wd = oracle.verify(LO, HI, p_fast=65521, dump=True)
    assert np.array_equal(d.cpu().numpy().astype(np.uint32), wd)
    for k in oracle.AGG_FIELDS:
        assert got[k] == want[k], (k, got[k], want[k])
    assert np.array_equal(np.asarray(got["hist"], dtype=np.int64), want["hist"])
    # the per-n kernel and single_check agree at the very top
    gp, dp = V.run(HI - 2**16, HI, dump=True, mode="pern")
    assert torch.equal(dp.cpu(), d[-dp.numel():].cpu())
    assert V.single_check(HI - 2) == int(wd[-1])
