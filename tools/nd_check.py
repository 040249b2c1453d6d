"""Device vs host nested dissection: identical permutation / ranges, timing.
    python tools/nd_check.py [grid nu n_a anchored] ..."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1104_3349_b200 as msc  # noqa: E402

cases = [(32, 0.1, 8, False), (128, 0.01, 16, False), (64, 0.002, 16, False),
         (256, 0.01, 64, False), (1024, 0.001, 1024, True)]
if len(sys.argv) > 1 and sys.argv[1] == "big":
    cases.append((2048, 0.01, 4096, True))
ctx = msc.Context(0)
msc.oseen_problem(8, 0.1, 2, ctx=ctx)  # warm the kernels
for g, nu, na, anch in cases:
    t0 = time.perf_counter()
    ph = msc.oseen_problem(g, nu, na, anchored=anch)
    t1 = time.perf_counter()
    pd = msc.oseen_problem(g, nu, na, anchored=anch, ctx=ctx)
    t2 = time.perf_counter()
    Ch, Cd = ph.C, pd.C
    same = (np.array_equal(ph.perm(), pd.perm()) and np.array_equal(ph.d_ranges(), pd.d_ranges())
            and np.array_equal(Ch.row_offsets, Cd.row_offsets)
            and np.array_equal(Ch.col_indices, Cd.col_indices)
            and np.array_equal(Ch.values.view(np.int64), Cd.values.view(np.int64))
            and ph.p == pd.p)
    print(f"grid {g} n_a {na}: host {t1 - t0:.3f} s, device {t2 - t1:.3f} s, identical {same}",
          flush=True)
    if not same:
        a, b = ph.perm(), pd.perm()
        d = np.nonzero(a != b)[0]
        print("  first diff at", d[:5], "ranges equal", np.array_equal(ph.d_ranges(), pd.d_ranges()),
              "nblocks", len(ph.d_ranges()), len(pd.d_ranges()))
