"""cfg4 apply with and without the split last wave (MSCG_TRI_NO_TAIL set in the
environment of the second run): writes the apply result for a bitwise
comparison and the D-solve time.

    python tools/tail_check.py out.npy
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    import paper_1104_3349_b200 as msc
    cfg = bench.CONFIGS[os.environ.get("CFG", "cfg4")]
    ctx = msc.Context(0)
    pb, _ = bench.build_problem(cfg, ctx=ctx)
    pc = msc.build_preconditioner(pb, tolA=bench.TOL_A, sA=bench.S_A, ctx=ctx)
    y = torch.from_numpy(bench.seeded_rhs(pb.n)).cuda()
    torch.cuda.synchronize()
    x = pc.apply(y)
    for _ in range(3):
        pc.apply(y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        x = pc.apply(y)
    torch.cuda.synchronize()
    print("apply ms", (time.perf_counter() - t0) / 20 * 1e3, flush=True)
    np.save(sys.argv[1], x.cpu().numpy())


if __name__ == "__main__":
    main()
