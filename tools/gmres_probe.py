"""Per-iteration cost of device GMRES vs its parts at one bench config.

    python tools/gmres_probe.py --config cfg4 --iters 200
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    import torch
    import bench
    import paper_1104_3349_b200 as msc
    from paper_1104_3349_b200.msc import SolverConfig
    cfg = bench.CONFIGS[a.config]
    ctx = msc.Context(0)
    pb, _ = bench.build_problem(cfg)
    pc = msc.build_preconditioner(pb, tolA=bench.TOL_A, sA=bench.S_A, ctx=ctx)
    b = torch.from_numpy(bench.seeded_rhs(pb.n)).cuda()
    out = {}
    for orth in ("cgs2", "mgs"):
        for its in (a.iters // 2, a.iters):
            scfg = SolverConfig(restart=cfg["restart"], max_iters=its, rel_tol=1e-8, orth=orth)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            msc.gmres(pc.matrix, pc, b, scfg)
            torch.cuda.synchronize()
            out[(orth, its)] = time.perf_counter() - t0
        per = (out[(orth, a.iters)] - out[(orth, a.iters // 2)]) / (a.iters - a.iters // 2)
        print(f"{orth}: {per * 1e3:.3f} ms per iteration (marginal, iterations "
              f"{a.iters // 2}..{a.iters})", flush=True)
    # the operator alone, synchronised like the Arnoldi loop
    x = torch.empty_like(b)
    y = torch.empty_like(b)
    for sync in (False, True):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(50):
            pc.apply_async(b.data_ptr(), x.data_ptr())
            if sync:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        print(f"apply loop (sync each={sync}): {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms",
              flush=True)


if __name__ == "__main__":
    main()
