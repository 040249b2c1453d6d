"""Summarise a trace written by tools/trace_dsolve.py (tiled kernel)."""
import sys

import numpy as np

z = np.load(sys.argv[1])
buf = z["trace"].astype(np.int64)
n = len(z["unnz"])
nt = (n + 31) // 32
t = buf[: 8 * nt].reshape(-1, 4)
base = t[0, 0]
t = t - base
solve = t[:, 2] - t[:, 1]
pw = t[:, 1] - t[:, 0]
dw = np.r_[0, t[1:, 0] - t[:-1, 3]]   # waiting for the tile's data
iss = t[:, 3] - t[:, 2]                # publish + TMA issue of a later tile
for nm, sl in (("L", slice(0, nt)), ("U", slice(nt, 2 * nt))):
    tot = t[sl][-1, 2] - (0 if nm == "L" else t[nt - 1, 2])
    print(nm, "tiles", nt, "total cyc", tot, "median solve", np.median(solve[sl]),
          "p90 solve", np.percentile(solve[sl], 90), "median part wait", np.median(pw[sl]),
          "median data wait", np.median(dw[sl]), "median issue", np.median(iss[sl]))
