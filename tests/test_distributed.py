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


def _shard_worker(rank, world, port, out):
    """One rank of a sharded interface exchange: F_r z_r over the rank's
    interior rows, summed by all-reduce, must equal F z."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch
    from paper_1104_3349_b200 import dist as d
    import paper_1104_3349_b200 as msc
    dist = d.init("gloo")
    pb = msc.oseen_problem(32, 0.1, 8)  # host setup layer only
    C = pb.C
    n, p = pb.n, pb.p
    dr = pb.d_ranges()
    b0, b1 = d.shard_blocks(dr[:, 1] - dr[:, 0], world)[rank]
    lo, hi = int(dr[b0, 0]), int(dr[b1 - 1, 1])
    z = np.random.default_rng(5).uniform(-1, 1, n)
    part = np.zeros(n - p)
    full = np.zeros(n - p)
    for i in range(p, n):
        s, e = C.row_offsets[i], C.row_offsets[i + 1]
        cols, vals = C.col_indices[s:e], C.values[s:e]
        m = cols < p
        full[i - p] = np.dot(vals[m], z[cols[m]])
        mr = (cols >= lo) & (cols < hi)
        part[i - p] = np.dot(vals[mr], z[cols[mr]])
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    out.put((rank, lo, hi, float(np.abs(t.numpy() - full).max()), float(np.abs(full).max())))
    dist.destroy_process_group()


def test_sharded_interface_exchange_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, lo0, hi0, e0, m0), (r1, lo1, hi1, e1, m1) = res
    assert lo0 == 0 and hi0 == lo1 and hi1 > lo1  # shards tile the interior rows
    assert e0 <= 1e-13 * m0 and e1 <= 1e-13 * m1
