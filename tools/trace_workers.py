"""Worker-time breakdown of a trace written by tools/trace_dsolve.py.

Per pass, sums over the 15 worker warps of block 0:
  need  - waiting for the item's input tiles (solver progress),
  dot   - loading + multiplying the item's far entries,
  pub   - waiting for a free slot in the partial-sum ring,
and the bytes each pass streamed, against the pass duration.
"""
import sys

import numpy as np

KW = 15
z = np.load(sys.argv[1])
buf = z["trace"].astype(np.int64)
n = len(z["unnz"])
nt = (n + 31) // 32
t = buf[: 8 * nt].reshape(-1, 4)
base = t[0, 0]
t = t - base
if "nitems" in z:
    last = int(z["nitems"])
    items = buf[8 * nt: 8 * nt + 4 * last].reshape(-1, 4)
else:
    items = buf[8 * nt:].reshape(-1, 4)
    valid = items[:, 0] != 0
    last = np.nonzero(valid)[0].max() + 1
    items = items[:last]
meta = items[:, 3]
need = meta >> 32
row = (meta & 0xffffffff) >> 3
st, de, pe = items[:, 0] - base, items[:, 1] - base, items[:, 2] - base
# split L / U lists: the U list starts where rows stop ascending from the tail
lrows = np.diff(row)
cut = np.nonzero(lrows < -40)[0]
nl = int(cut[0]) + 1 if len(cut) else last
for name, sl, q0 in (("L", slice(0, nl), 0), ("U", slice(nl, last), nt)):
    s, d, p, nd = st[sl], de[sl], pe[sl], need[sl]
    if len(s) == 0:
        continue
    ready = np.where(nd > 0, t[np.clip(q0 + nd - 1, 0, 2 * nt - 1), 2], 0)
    wait_need = np.clip(ready - s, 0, None)
    dot = d - np.maximum(s, ready)
    pub = p - d
    p0 = 0 if name == "L" else t[nt - 1, 2]
    p1 = t[nt - 1, 2] if name == "L" else t[2 * nt - 1, 2]
    dur = p1 - p0
    busy = KW * dur
    print(f"{name}: pass {dur} cyc, {len(s)} items; worker time share: need "
          f"{wait_need.sum() / busy:.2f} dot {dot.sum() / busy:.2f} pub {pub.sum() / busy:.2f}"
          f" idle {1 - (wait_need.sum() + dot.sum() + pub.sum()) / busy:.2f}; median dot "
          f"{np.median(dot):.0f} cyc")
    # coarse timeline: fraction of workers computing per 1/10 of the pass
    edges = np.linspace(p0, p1, 11)
    occ = []
    for a, b in zip(edges[:-1], edges[1:]):
        lo, hi = np.maximum(np.maximum(s, ready), a), np.minimum(d, b)
        occ.append(np.clip(hi - lo, 0, None).sum() / (KW * (b - a)))
    print("   computing fraction per tenth:", " ".join(f"{o:.2f}" for o in occ))
