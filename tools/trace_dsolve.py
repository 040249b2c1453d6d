"""Timing trace of the interior-block triangular solve (block 0).

    python tools/trace_dsolve.py --config cfg2 [--out gpurun_out/trace_cfg2.npz]

Stores the raw clock64 stamps of block 0 (solver: per tile [data ready, far
sums ready, tile solved] for the L then U stream; workers: per row [start,
far dot done, published] at offset 6*ntiles) plus block 0's factor row
lengths, for offline analysis with tools/trace_tiles.py.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import bench
    import paper_1104_3349_b200 as msc
    from paper_1104_3349_b200 import _capi
    cfg = bench.CONFIGS[a.config]
    ctx = msc.Context(0)
    pb, _ = bench.build_problem(cfg)
    pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
    y = torch.from_numpy(bench.seeded_rhs(pb.n)).cuda()
    x = torch.empty_like(y)
    torch.cuda.synchronize()
    f = pc.d_factors(0)
    n = f.upper.nrows
    buf = np.zeros(32 * n, np.int64)
    st = _capi.Status()
    for _ in range(3):  # warm
        rc = _capi.lib().mscg_debug_trace_dsolve(pc.h, C.c_void_p(y.data_ptr()),
                                                 C.c_void_p(x.data_ptr()),
                                                 buf.ctypes.data_as(C.c_void_p), 32 * n,
                                                 C.byref(st))
    assert rc == n, (rc, st.message)
    out = a.out or os.path.join(ROOT, "gpurun_out", f"trace_{a.config}.npz")
    # far work items of block 0, as factor.cu's pack kernel builds them: long
    # rows in kSeg = 512 pieces (at most 4), runs of short rows (<= 96
    # entries) of one tile grouped up to 128 entries.  The trace holds 4
    # stamps per item.
    def nitems(m, lower):
        rp, ci = m.row_offsets, m.col_indices
        cnt = []
        for i in range(n):
            c = ci[rp[i]:rp[i + 1]]
            t = i // 32
            cnt.append(int((c < 32 * (t - 2)).sum()) if lower else int((c >= 32 * (t + 3)).sum()))
        order = range(n) if lower else range(n - 1, -1, -1)
        tot, g0, g1, gent = 0, -1, -1, 0
        for i in order:
            c = cnt[i]
            if c == 0:
                continue
            if c <= 96:
                if g0 >= 0:
                    lo, hi = min(g0, i), max(g1, i)
                    if i // 32 != g0 // 32 or gent + c > 128 or hi - lo >= 32:
                        tot += 1
                        g0 = -1
                if g0 < 0:
                    g0 = g1 = i
                    gent = 0
                else:
                    g0, g1 = min(g0, i), max(g1, i)
                gent += c
                continue
            if g0 >= 0:
                tot += 1
                g0 = -1
            tot += min(4, (c + 511) // 512)
        if g0 >= 0:
            tot += 1
        return tot
    np.savez_compressed(out, trace=buf, lnnz=np.diff(f.lower.row_offsets),
                        unnz=np.diff(f.upper.row_offsets),
                        nitems=nitems(f.lower, True) + nitems(f.upper, False))
    print("trace written to", out)


if __name__ == "__main__":
    main()
