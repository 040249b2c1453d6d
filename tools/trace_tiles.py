"""Summarise a per-tile trace from tools/trace_dsolve.py (tiled kernel)."""
import sys
import numpy as np
z = np.load(sys.argv[1]); tr = z['trace'].reshape(-1, 3)
n = len(z['unnz']); nt = (n + 31) // 32
t = tr[:2 * nt].astype(np.int64); t = t - t[0, 0]
solve = t[:, 2] - t[:, 1]; pw = t[:, 1] - t[:, 0]
dw = np.r_[0, t[1:, 0] - t[:-1, 2]]
for nm, sl in (("L", slice(0, nt)), ("U", slice(nt, 2 * nt))):
    print(nm, "tiles", nt, "total", t[sl][-1, 2] - (t[sl][0, 0] if nm == "L" else t[nt - 1, 2]),
          "median solve", np.median(solve[sl]), "p90 solve", np.percentile(solve[sl], 90),
          "median part wait", np.median(pw[sl]), "p90", np.percentile(pw[sl], 90),
          "median data wait", np.median(dw[sl]))
print("slow tiles (solve > 5000):", np.nonzero(solve > 5000)[0][:40])
