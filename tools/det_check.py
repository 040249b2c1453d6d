import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_1104_3349_b200 as msc
from paper_1104_3349_b200 import dist
ctx = msc.Context(0)
pb = msc.oseen_problem(128, 0.01, 16); pb.build_msc("lum")
full = msc.build_preconditioner(pb, tolA=1e-4, sA=0, ctx=ctx)
y = np.random.default_rng(1).uniform(-1, 1, pb.n)
a = full.apply(y); b = full.apply(y)
print("full apply deterministic:", np.array_equal(a.view(np.int64), b.view(np.int64)), np.abs(a-b).max())
n, p = pb.n, pb.p
dr = pb.d_ranges()
ranges = dist.shard_blocks(dr[:, 1] - dr[:, 0], 2)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
shards = [msc.build_preconditioner_shard(pb, b0, b1, tolA=1e-4, sA=0, ctx=ctx) for b0, b1 in ranges]
yd = torch.from_numpy(y).cuda()
ts = [torch.empty(n - p, dtype=torch.float64, device="cuda") for _ in shards]
for s, t in zip(shards, ts): s.apply_begin(yd, t)
tsum = torch.stack(ts).sum(0)
outs = []
for rep in range(2):
    for s in shards:
        x = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
        s.apply_end(yd, tsum, x)
        outs.append(x[p:].cpu().numpy())
for o in outs[1:]:
    print("x2 equal to first:", np.array_equal(o, outs[0]), np.abs(o - outs[0]).max())
# Schur factors of shard 0 vs full
for k in range(3):
    f0 = full.schur_factors(k)
print("ts nan:", [int(torch.isnan(t).sum()) for t in ts], "tsum nan:", int(torch.isnan(tsum).sum()))
for k, o in enumerate(outs):
    bad = np.nonzero(np.isnan(o))[0]
    print("out", k, "nan count", len(bad), bad[:10])
# unsharded reference pieces
xf = full.apply(yd)  # device path
xf = xf.cpu().numpy()
xh = full.apply(y)   # host path
print("full device vs host path equal:", np.array_equal(xf, xh), "nan", np.isnan(xf).sum(), np.isnan(xh).sum())
print("x2 shard vs full max diff:", np.abs(outs[0] - xf[p:]).max(), "scale", np.abs(xf[p:]).max())
# interior rows from the shards
got = np.full(n, np.nan)
for s in shards:
    x = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    s.apply_end(yd, tsum, x)
    lo, hi = s.rows
    got[lo:hi] = x[lo:hi].cpu().numpy()
got[p:] = outs[0]
print("interior nan:", np.isnan(got[:p]).sum(), "interior max diff:", np.nanmax(np.abs(got[:p] - xf[:p])))
