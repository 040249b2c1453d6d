"""Worker-item view of a trace written by tools/trace_dsolve.py (v4 kernel)."""
import sys

import numpy as np

z = np.load(sys.argv[1])
buf = z["trace"].astype(np.int64)
n = len(z["unnz"])
nt = (n + 31) // 32
t = buf[: 6 * nt].reshape(-1, 3)
base = t[0, 0]
items = buf[6 * nt:].reshape(-1, 4)
m = items[:, 0] != 0
it = items[m]
print("items traced", m.sum())
st = it[:, 0] - base
dot = it[:, 1] - it[:, 0]
pub = it[:, 2] - it[:, 1]
row = it[:, 3] >> 3
seg = it[:, 3] & 7
order = np.argsort(st)
print("median dot", np.median(dot), "p90", np.percentile(dot, 90), "median publish", np.median(pub))
for k in list(range(0, len(it), max(1, len(it) // 40))):
    q = order[k]
    print(f"start {st[q]:9d} dot {dot[q]:7d} pub {pub[q]:6d} row {row[q]:5d} tile {row[q] // 32:3d} seg {seg[q]}")
