"""TEST INFRASTRUCTURE: one rank of the 2-process sharded solve, launched by
tests/test_gpu_dist.py through torchrun (gloo on CUDA tensors; both ranks
share the box's one GPU — a functional check of the N>1 path, never a
timing).  Each rank builds its shard of the cfg1 preconditioner and, for the
check, the whole preconditioner; rank 0 prints one JSON line."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import paper_1104_3349_b200 as msc
    from paper_1104_3349_b200 import dist as pdist
    from paper_1104_3349_b200 import _capi

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    ctx = msc.Context(0)
    grid, nu, n_a = (int(os.environ.get("DW_GRID", "32")), float(os.environ.get("DW_NU", "0.1")),
                     int(os.environ.get("DW_NA", "8")))
    pb = msc.oseen_problem(grid, nu, n_a)
    pb.build_msc("lum")
    dr = pb.d_ranges()
    b0, b1 = pdist.shard_blocks(dr[:, 1] - dr[:, 0], world)[rank]
    sh = msc.build_preconditioner_shard(pb, b0, b1, tolA=1e-4, sA=0, ctx=ctx)
    full = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    n, p = pb.n, pb.p
    ng = n - p
    lo, hi = sh.rows
    own = np.r_[lo:hi, p:n]
    dev = torch.device("cuda", 0)
    torch.cuda.synchronize()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)

    def rel(a, b):
        return float(np.linalg.norm(a - b) / np.linalg.norm(b))

    # one preconditioner apply across the processes
    y = np.random.default_rng(3).uniform(-1, 1, n)
    yd = torch.from_numpy(y).to(dev)
    xd = torch.zeros(n, dtype=torch.float64, device=dev)
    t = torch.zeros(max(ng, 1), dtype=torch.float64, device=dev)
    sh.apply_begin(yd, t)
    dist.all_reduce(t)
    sh.apply_end(yd, t, xd)
    x_apply = xd.cpu().numpy()
    want = full.apply(y)
    err_apply = rel(x_apply[own], want[own])

    # one matvec of C across the processes
    w = torch.zeros(n, dtype=torch.float64, device=dev)
    y2 = torch.zeros(max(ng, 1), dtype=torch.float64, device=dev)
    sh.spmv(yd, w, y2, rank == 0)
    dist.all_reduce(y2)
    got = np.concatenate([w.cpu().numpy()[lo:hi], y2.cpu().numpy()[:ng]])
    want_mv = msc.matvec(full.matrix, y)
    err_spmv = rel(got, want_mv[own])

    # distributed GMRES (DCGS2) vs the single-GPU solve of the same system
    b = np.empty(n)
    _capi.lib().mscg_random_vector(n, 0, b.ctypes.data_as(_capi.C.c_void_p))
    cfg = msc.SolverConfig(restart=30, max_iters=3000, rel_tol=1e-8, orth="dcgs2")
    x, rep = sh.gmres(b, cfg, rank, world)
    ctx.set_stream(None)
    x1, rep1 = msc.gmres(full.matrix, full, b, cfg)
    xa = torch.from_numpy(np.where(np.arange(n) < p, x, x if rank == 0 else 0.0))
    dist.all_reduce(xa)
    xa = xa.numpy()
    tr = msc.true_residual(full.matrix, xa, b)
    h0, h1 = np.asarray(rep.residual_history), np.asarray(rep1.residual_history)
    k = min(len(h0), len(h1)) - 1
    out = {"rank": rank, "world": world, "rows": [int(lo), int(hi)], "blocks": [int(b0), int(b1)],
           "err_apply": err_apply, "err_spmv": err_spmv,
           "its": rep.iterations, "its_single": rep1.iterations, "converged": rep.converged,
           "true_residual": tr, "hist_dev": float(np.max(np.abs(h0[:k] - h1[:k]) / np.abs(h1[:k]))),
           "x_rel": rel(xa, x1)}
    outs = [None] * world
    dist.all_gather_object(outs, out)
    if rank == 0:
        print("DIST_RESULT " + json.dumps(outs), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
