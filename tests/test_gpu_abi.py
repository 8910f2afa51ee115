"""The C ABI's host entry point, launch accounting and error contract on a GPU
(include/gb.h): gb_verify_range_host against the oracle (its dump is moved through
the ctx scratch in 2^24-even chunks), one launch per plain gb_verify_range, and the
documented error statuses."""
import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def V():
    from paper_2603_02621_b200.verifier import Verifier
    v = Verifier(hi_max=10**9 + 1, p_max=65521)
    yield v
    v.close()


def test_host_entry_point_vs_oracle(V):
    from paper_2603_02621_b200 import gb
    lo, hi = 10**9 - 2**25 - 1234, 10**9 + 1          # > 2^24 evens: two dump chunks
    n = (hi - (lo + (lo & 1)) + 1) // 2
    h_res = torch.empty(gb.RESULT_WORDS, dtype=torch.int64).pin_memory()
    h_dump = np.zeros(n, dtype=np.uint32)
    gb.gb_verify_range_host(V.ctx, lo, hi, 65521, h_res, h_dump, V.stream)
    got = gb.decode_result(h_res)
    want, wd = oracle.verify(lo, hi, p_fast=65521, dump=True)
    assert np.array_equal(h_dump, wd)
    for k in oracle.AGG_FIELDS:
        assert got[k] == want[k], k
    assert np.array_equal(np.asarray(got["hist"]), want["hist"])


def test_one_launch_per_verify(V):
    from paper_2603_02621_b200 import gb
    r = V.new_result()
    c0 = gb.gb_launch_count()
    V.verify(4, 10**8 + 1, r)
    assert gb.gb_launch_count() - c0 == 1
    V.verify(10, 10, r)                                  # empty range: no launch
    assert gb.gb_launch_count() - c0 == 1


def test_error_contract(V):
    from paper_2603_02621_b200 import gb
    r = V.new_result()
    cases = [
        (lambda: gb.gb_verify_range(V.ctx, 100, 50, 65521, r, None, V.stream), gb.GB_EINVAL),      # lo > hi
        (lambda: gb.gb_verify_range(V.ctx, 4, 10**9 + 3, 65521, r, None, V.stream), gb.GB_ERANGE),  # > hi_max
        (lambda: gb.gb_verify_range(V.ctx, 4, 1000, 2, r, None, V.stream), gb.GB_EINVAL),          # p_max < 3
        (lambda: gb.gb_verify_range(V.ctx, 4, 1000, 65537, r, None, V.stream), gb.GB_EINVAL),      # > ctx p_max
        (lambda: gb.gb_single_check(V.ctx, 7, 100, r, V.stream), gb.GB_EINVAL),                    # odd n
    ]
    for f, st in cases:
        with pytest.raises(gb.GBError) as e:
            f()
        assert e.value.status == st
    # a workspace one byte short is refused before any device work
    need = gb.gb_ctx_workspace_bytes(10**7, 65521)
    ws = torch.empty(need - 256, dtype=torch.uint8, device=V.device)
    with pytest.raises(gb.GBError) as e:
        gb.gb_ctx_create(V.device.index, 0, 10**7, 65521, ws, V.stream)
    assert e.value.status == gb.GB_EWORKSPACE
    # counterexample is a result, not an error: capped fallback leaves n unresolved
    got, _ = V.run(4, 10**4 + 1, p_max=3, cap=5)
    assert got["unresolved"] > 0 and got["first_unresolved_n"] >= 4
