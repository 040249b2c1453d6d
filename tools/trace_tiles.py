"""Summarise a trace written by tools/trace_dsolve.py (tiled kernel)."""
import sys

import numpy as np

z = np.load(sys.argv[1])
buf = z["trace"].astype(np.int64)
n = len(z["unnz"])
nt = (n + 31) // 32
t = buf[: 6 * nt].reshape(-1, 3)
base = t[0, 0]
t = t - base
solve = t[:, 2] - t[:, 1]
pw = t[:, 1] - t[:, 0]
dw = np.r_[0, t[1:, 0] - t[:-1, 2]]
for nm, sl in (("L", slice(0, nt)), ("U", slice(nt, 2 * nt))):
    tot = t[sl][-1, 2] - (0 if nm == "L" else t[nt - 1, 2])
    print(nm, "tiles", nt, "total cyc", tot, "median solve", np.median(solve[sl]),
          "p90 solve", np.percentile(solve[sl], 90), "median part wait", np.median(pw[sl]),
          "median data wait", np.median(dw[sl]))
rows = buf[6 * nt: 6 * nt + 6 * n].reshape(2, n, 3)
for k, nm in ((0, "L"), (1, "U")):
    r = rows[k]
    m = r[:, 0] != 0
    if not m.any():
        continue
    r = r[m] - base
    idx = np.nonzero(m)[0]
    nn = (z["lnnz"] if k == 0 else z["unnz"])[idx]
    dot = r[:, 1] - r[:, 0]
    pub = r[:, 2] - r[:, 1]
    print(f"{nm} workers: rows with far entries {m.sum()}, median dot {np.median(dot):.0f} cyc "
          f"(p90 {np.percentile(dot, 90):.0f}), median publish wait {np.median(pub):.0f}, "
          f"median row nnz {np.median(nn):.0f}")
    # per-tile: when was the last far sum of the tile published vs tile solved
    tiles = idx // 32
    for tt in sorted(set(tiles))[:: max(1, len(set(tiles)) // 12)]:
        sel = tiles == tt
        q = tt if k == 0 else nt + (nt - 1 - tt)
        print(f"   tile {tt}: rows {sel.sum()} first start {r[sel, 0].min()} last pub "
              f"{r[sel, 2].max()}  solver data {t[q, 0]} solved {t[q, 2]}")
