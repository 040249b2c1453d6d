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


# ---- the distributed DCGS2 GMRES decomposition (csrc/device/gmres.cu,
# gmres_shard) restated in numpy: compact per-rank vectors [own interior
# rows | interface], the interface replicated, dots counting it on rank 0
# only, two all-reduces per Arnoldi step plus the operator's two.  Run under
# gloo with 2 processes and compared with the single-process restatement.

def _dcgs2_gmres(op, dot, b, m, tol, maxit):
    """Right-preconditioned restarted GMRES with DCGS2 (the device algorithm,
    restated); `op` applies A B^-1, `dot` is the (global) inner product of
    two local vectors.  Returns (x_krylov_combination, its, history)."""
    n = len(b)
    nrm = lambda v: np.sqrt(dot(v, v))
    x = np.zeros(n)
    denom = nrm(b)
    hist, its = [], 0
    while True:
        r = b - op["A"](x)
        beta = nrm(r)
        if not hist:
            hist.append(beta / denom)
        if beta / denom <= tol:
            break
        V = np.zeros((m + 1, n))
        V[0] = r
        nu = np.zeros(m + 2)
        nu[0] = beta
        Hraw = np.zeros((m + 1, m))
        R = np.zeros((m + 1, m))
        cs, sn = np.zeros(m + 1), np.zeros(m + 1)
        g = np.zeros(m + 2)
        g[0] = beta

        def rotate(col, k):
            for i in range(k):
                t1 = cs[i] * col[i] + sn[i] * col[i + 1]
                col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
                col[i] = t1
            dr = np.hypot(col[k], col[k + 1])
            return (1.0, 0.0) if dr == 0 else (col[k] / dr, col[k + 1] / dr)

        def fix(j, w):
            y = V[j]
            s = np.array([dot(V[i], y) for i in range(j)]) / nu[j]
            rho = 1.0
            if j > 0:
                rho = np.sqrt(dot(y, y) / nu[j] ** 2 - s @ s)
                Hraw[:j, j - 1] += nu[j] * s
                Hraw[j, j - 1] = nu[j] * rho
                col = Hraw[:j + 1, j - 1].copy()
                cs[j - 1], sn[j - 1] = rotate(col, j - 1)
                R[:j + 1, j - 1] = col
                g[j] = -sn[j - 1] * g[j - 1]
                g[j - 1] = cs[j - 1] * g[j - 1]
            if w is None:
                return None
            t = np.array([dot(V[i], w) for i in range(j)]) / nu[j]
            c = (dot(y, w) / nu[j] ** 2 - s @ t) / rho
            Hraw[:j + 1, j] = (np.append(t, c) - Hraw[:j + 1, :j] @ s) / rho
            return s, t, c, rho

        jmax = min(m, maxit - its)
        mm = 0
        for j in range(jmax):
            w = op["AB"](V[j])
            s, t, c, rho = fix(j, w)
            q = (V[j] / nu[j] - V[:j].T @ s) / rho
            V[j + 1] = (w / nu[j] - V[:j].T @ t - c * q) / rho
            V[j] = q
            nu[j + 1] = nrm(V[j + 1])
            Hraw[j + 1, j] = nu[j + 1]
            col = Hraw[:j + 2, j].copy()
            _, s_ = rotate(col, j)
            its += 1
            mm = j + 1
            hist.append(abs(-s_ * g[j]) / denom)
            if hist[-1] <= tol:
                break
        fix(mm, None)
        y = np.zeros(mm)
        for i in range(mm - 1, -1, -1):
            y[i] = (g[i] - R[i, i + 1:mm] @ y[i + 1:mm]) / R[i, i]
        x = x + op["B"](V[:mm].T @ y)
        if nrm(b - op["A"](x)) / denom <= tol or its >= maxit:
            break
    return x, its, hist


def _saddle_system(n_blocks=4, bs=30, ng=12, seed=3):
    """Block-diagonal interior + interface coupling, as the MSC split has it."""
    rng = np.random.default_rng(seed)
    p = n_blocks * bs
    n = p + ng
    A = np.zeros((n, n))
    for k in range(n_blocks):
        sl = slice(k * bs, (k + 1) * bs)
        A[sl, sl] = np.eye(bs) * 4 + rng.uniform(-1, 1, (bs, bs)) * 0.3
    A[:p, p:] = rng.uniform(-1, 1, (p, ng)) * (rng.uniform(size=(p, ng)) < 0.2)
    A[p:, :p] = rng.uniform(-1, 1, (ng, p)) * (rng.uniform(size=(ng, p)) < 0.2)
    A[p:, p:] = np.eye(ng) * 3
    b = rng.uniform(-1, 1, n)
    # preconditioner: block Jacobi on the interior blocks, identity on the interface
    Binv = np.zeros((n, n))
    for k in range(n_blocks):
        sl = slice(k * bs, (k + 1) * bs)
        Binv[sl, sl] = np.linalg.inv(A[sl, sl])
    Binv[p:, p:] = np.eye(ng)
    return A, Binv, b, p, bs


def _dist_gmres_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch
    from paper_1104_3349_b200 import dist as d
    dist = d.init("gloo")
    A, Binv, b, p, bs = _saddle_system()
    n = len(b)
    nb = p // bs
    b0, b1 = d.shard_blocks([bs] * nb, world)[rank]
    lo, hi = b0 * bs, b1 * bs
    own = np.r_[lo:hi, p:n]  # compact layout: own interior rows | interface

    def allsum(v):
        t = torch.from_numpy(np.ascontiguousarray(v, np.float64).copy())
        dist.all_reduce(t)
        return t.numpy()

    def dot(u, v):  # interface counted on rank 0 only
        k = hi - lo + (n - p if rank == 0 else 0)
        return float(allsum(np.array([u[:k] @ v[:k]]))[0])

    def to_global(c):
        gv = np.zeros(n)
        gv[own] = c
        return gv

    def op_A(c):  # interior rows of C need only own + interface columns
        gv = to_global(c)
        y1 = A[lo:hi] @ gv
        y2 = allsum(A[p:, lo:hi] @ gv[lo:hi] + (A[p:, p:] @ gv[p:] if rank == 0 else 0.0))
        return np.concatenate([y1, y2])

    def op_B(c):
        gv = to_global(c)
        return np.concatenate([Binv[lo:hi, lo:hi] @ gv[lo:hi], gv[p:]])

    op = {"A": op_A, "B": op_B, "AB": lambda c: op_A(op_B(c))}
    x, its, hist = _dcgs2_gmres(op, dot, b[own], 10, 1e-10, 300)
    out.put((rank, its, list(hist), x.tolist(), own.tolist()))
    dist.destroy_process_group()


def test_distributed_dcgs2_gmres_decomposition_gloo():
    """The decomposition gmres_shard uses, restated in numpy and run on two
    gloo ranks, equals the single-process DCGS2 solve: same iterations,
    residual histories to 1e-10, and the assembled solution solves A x = b."""
    import torch.multiprocessing as mp
    A, Binv, b, p, bs = _saddle_system()
    n = len(b)
    single = {"A": lambda v: A @ v, "B": lambda v: Binv @ v, "AB": lambda v: A @ (Binv @ v)}
    x1, its1, hist1 = _dcgs2_gmres(single, lambda u, v: float(u @ v), b, 10, 1e-10, 300)
    assert np.linalg.norm(b - A @ x1) / np.linalg.norm(b) <= 1e-10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_gmres_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    x = np.zeros(n)
    for rank, its, hist, xl, own in res:
        assert its == its1
        assert np.allclose(hist, hist1, rtol=1e-10, atol=1e-14)
        xl = np.asarray(xl)
        own = np.asarray(own)
        interior = own < p
        x[own[interior]] = xl[interior]
        if rank == 0:
            x[own[~interior]] = xl[~interior]
    assert np.linalg.norm(x - x1) <= 1e-9 * np.linalg.norm(x1)
