"""Per-step wall times of the host-buffer (C ABI) step at cfg5: apply + SpMV.

    python tools/e2e_steps.py [steps]
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1104_3349_b200 as msc
from paper_1104_3349_b200 import _capi

n_steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
L = _capi.lib()
ctx = msc.Context(0)
pb, _ = bench.build_problem(bench.CONFIGS["cfg5"], ctx=ctx)
pc = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
y = torch.from_numpy(bench.seeded_rhs(pb.n)).pin_memory()
x = torch.empty(pb.n, dtype=torch.float64).pin_memory()
w = torch.empty(pb.n, dtype=torch.float64).pin_memory()
mat = L.mscg_precond_matrix(pc.h)
st = _capi.Status()
ts = []
for _ in range(n_steps):
    t0 = time.perf_counter()
    L.mscg_precond_apply(pc.h, C.c_void_p(y.data_ptr()), C.c_void_p(x.data_ptr()), _capi.MEM_HOST,
                         C.byref(st))
    t1 = time.perf_counter()
    L.mscg_spmv(mat, C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), _capi.MEM_HOST,
                C.byref(st))
    t2 = time.perf_counter()
    ts.append((1e3 * (t1 - t0), 1e3 * (t2 - t1)))
print("apply ms:", " ".join(f"{a:.2f}" for a, _ in ts))
print("spmv  ms:", " ".join(f"{b:.2f}" for _, b in ts))
