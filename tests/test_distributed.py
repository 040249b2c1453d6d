"""CPU: the N>1 plumbing (world_size 2, gloo backend, 127.0.0.1)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_1104_3349_b200 import dist as d
    dist = d.init("gloo")
    ws, r, lr = d.env()
    # each rank "times" a different duration; the report is the max
    t = d.max_over_ranks(10.0 + 5.0 * rank, dist)
    dist.barrier()
    out.put((rank, ws, r, t))
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] == 2 for r in res)
    assert all(r[3] == 15.0 for r in res)


def test_bench_replica_line_under_gloo_launch(tmp_path):
    """bench.py's multi-rank aggregation: value = total steps of all ranks /
    max time.  Exercised through the same helper the bench uses."""
    from paper_1104_3349_b200 import dist as d
    assert d.max_over_ranks(3.5) == 3.5


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_blocks_covers_all_blocks(world):
    from paper_1104_3349_b200 import dist as d
    rows = np.random.default_rng(1).integers(2500, 3400, 64)
    sh = d.shard_blocks(rows, world)
    assert len(sh) == world
    assert sh[0][0] == 0 and sh[-1][1] == 64
    for (a, b), (c, e) in zip(sh, sh[1:]):
        assert b == c and a <= b
    sizes = [rows[a:b].sum() for a, b in sh]
    assert max(sizes) - min(sizes) <= 2 * rows.max()
