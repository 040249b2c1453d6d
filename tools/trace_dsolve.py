"""Per-row timing trace of the interior-block triangular solve (block 0).

    python tools/trace_dsolve.py --config cfg2 --out gpurun_out/trace_cfg2.npz

Stores clock64 stamps (row start, head reduced, row published) for the L and
U sweeps plus block 0's factor row lengths, for offline analysis.
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
    buf = np.zeros(6 * n, np.int64)
    st = _capi.Status()
    for _ in range(3):  # warm
        rc = _capi.lib().mscg_debug_trace_dsolve(pc.h, C.c_void_p(y.data_ptr()),
                                                 C.c_void_p(x.data_ptr()),
                                                 buf.ctypes.data_as(C.c_void_p), 6 * n,
                                                 C.byref(st))
    assert rc == n, (rc, st.message)
    tr = buf.reshape(2, n, 3)
    t0 = tr[0, :, 0].min()
    tr = tr - t0
    lnnz = np.diff(f.lower.row_offsets)
    unnz = np.diff(f.upper.row_offsets)
    out = a.out or os.path.join(ROOT, "gpurun_out", f"trace_{a.config}.npz")
    np.savez_compressed(out, trace=tr, lnnz=lnnz, unnz=unnz)
    for k, nm in ((0, "L"), (1, "U")):
        t = tr[k]
        span = t[:, 2].max() - t[:, 0].min()
        print(f"{nm}: rows {n} span {span} cyc ({span / 1.9e3:.1f} us @1.9GHz); "
              f"median row latency {np.median(t[:, 2] - t[:, 0]):.0f} cyc, "
              f"median head {np.median(t[:, 1] - t[:, 0]):.0f} cyc")


if __name__ == "__main__":
    main()
