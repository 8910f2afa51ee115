"""The N > 1 path through libgb on one GPU: ranks sharing cuda:0 over a gloo
process group (NCCL refuses two ranks on one device; the round-end boxes have one
GPU).  Each rank verifies its round-robin strips of [4, 1e10] with
gb_verify_range, finalizes, and dist.reduce_result combines the result vectors
(SUM / MAX / MIN); rank 0's reduced vector must equal the oracle golden
(tests/golden/verify_1e10.json) field by field.  Also bench.py under torchrun with
2 ranks, whose own golden check must pass (section 3.5)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from oracle import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
mp = pytest.importorskip("torch.multiprocessing")

N = 10**10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_02621_b200 import dist as gdist
    from paper_2603_02621_b200.verifier import Verifier
    v = Verifier(hi_max=N + 1)
    r = gdist.verify_sharded(v, 4, N + 1, rank, world, strips_per_rank=4)
    torch.cuda.synchronize()
    if rank == 0:
        q.put(v.decode(r))
    dist.barrier()
    v.close()
    dist.destroy_process_group()


def _golden():
    g = json.load(open(os.path.join(GOLDEN, "verify_1e10.json")))
    assert (g["lo"], g["hi"]) == (4, N + 1)
    return g["result"]


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_share_gpu_match_golden(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = _golden()
    for k in oracle.AGG_FIELDS:
        assert got[k] == g[k], (k, got[k], g[k])
    hist = np.zeros(oracle.NBINS, np.int64)
    for i, c in g["hist"].items():
        hist[int(i)] = c
    assert np.array_equal(np.asarray(got["hist"]), hist)


def test_bench_two_ranks_torchrun():
    env = dict(os.environ, GB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--N", "1e10", "--steps", "1", "--warmup", "3",
           "--no-cpu-baseline", "--no-sieve"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["check"]["ok"] and line["check"]["golden"]
    assert line["result"]["evens"] == N // 2 - 1
