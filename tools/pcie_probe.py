"""Host-buffer path costs at cfg5: raw H2D/D2H of one vector, host-buffer apply and SpMV, device apply.

    python tools/pcie_probe.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, json
import bench, paper_1104_3349_b200 as msc
import ctypes as C
from paper_1104_3349_b200 import _capi
L=_capi.lib()
ctx=msc.Context(0)
pb,_=bench.build_problem(bench.CONFIGS['cfg5'], ctx=ctx)
pc=msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
n=pb.n
y=torch.from_numpy(bench.seeded_rhs(n,0)).pin_memory(); x=torch.empty(n,dtype=torch.float64).pin_memory(); w=torch.empty(n,dtype=torch.float64).pin_memory()
d=torch.empty(n,dtype=torch.float64,device='cuda')
mat=L.mscg_precond_matrix(pc.h)
def t(f,k=10):
    f(); torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/k*1e3
st=_capi.Status()
print("H2D 100MB ms", t(lambda: d.copy_(y, non_blocking=True)))
print("D2H 100MB ms", t(lambda: x.copy_(d, non_blocking=True)))
print("apply host ms", t(lambda: L.mscg_precond_apply(pc.h, C.c_void_p(y.data_ptr()), C.c_void_p(x.data_ptr()), _capi.MEM_HOST, C.byref(st))))
print("spmv host ms", t(lambda: L.mscg_spmv(mat, C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), _capi.MEM_HOST, C.byref(st))))
yd=y.cuda(); xd=torch.empty_like(yd)
print("apply dev ms", t(lambda: pc.apply_async(yd.data_ptr(), xd.data_ptr())))
