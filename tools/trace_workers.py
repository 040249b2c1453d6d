"""Worker-side view of a trace written by tools/trace_dsolve.py (block 0).

Per pass: items, their busy time (from the later of start and readiness to
the end of the dot), the workers' busy fraction per twentieth of the pass and
the distribution of `need`.  The U items are those started after the L pass
ended.

    python tools/trace_workers.py gpurun_out/trace_cfg5.npz [workers=15]
"""
import sys

import numpy as np

KW = int(sys.argv[2]) if len(sys.argv) > 2 else 15
z = np.load(sys.argv[1])
buf = z["trace"].astype(np.int64)
n = len(z["unnz"])
nt = (n + 31) // 32
t = buf[: 8 * nt].reshape(-1, 4)
base = t[0, 0]
t = t - base
items = buf[8 * nt:].reshape(-1, 4)
valid = np.nonzero(items[:, 0] != 0)[0]
it = items[: valid.max() + 1]
meta = it[:, 3]
need = meta >> 32
st, de = it[:, 0] - base, it[:, 1] - base
l_end = t[nt - 1, 2]
nl = int(np.nonzero(st >= l_end - 1000)[0][0])
print(f"L pass {l_end} cycles, U pass {t[2 * nt - 1, 2] - l_end}; items L {nl} U {len(it) - nl}")
for name, sl, q0 in (("L", slice(0, nl), 0), ("U", slice(nl, len(it)), nt)):
    s, d, nd = st[sl], de[sl], need[sl]
    if len(s) == 0:
        continue
    ready = np.where(nd > 0, t[np.clip(q0 + nd - 1, 0, 2 * nt - 1), 2], 0)
    busy = d - np.maximum(ready, s)
    print(f"{name}: {len(s)} items, busy median {np.median(busy):.0f} mean {busy.mean():.0f} cycles, "
          f"sum/{KW} workers {busy.sum() / KW:.0f}; started after ready by median "
          f"{np.median(s - ready):.0f} cycles")
    p0 = 0 if name == "L" else l_end
    p1 = l_end if name == "L" else t[2 * nt - 1, 2]
    edges = np.linspace(p0, p1, 21)
    occ = []
    for a, b in zip(edges[:-1], edges[1:]):
        lo, hi = np.maximum(np.maximum(s, ready), a), np.minimum(d, b)
        occ.append(np.clip(hi - lo, 0, None).sum() / (KW * (b - a)))
    print("   busy fraction per 1/20:", " ".join(f"{o:.2f}" for o in occ))
    print("   need quantiles (0,10,25,50,75,90,100 %):",
          np.percentile(nd, [0, 10, 25, 50, 75, 90, 100]).astype(int).tolist())
