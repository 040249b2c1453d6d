"""Count solver stalls in a trace (tools/trace_dsolve.py): tiles whose 32-row
chain took > 8K cycles, and tiles whose far sums arrived > 8K cycles after
the tile landed although every work item of the tile had been published
before it landed."""
import sys

import numpy as np

z = np.load(sys.argv[1])
buf = z["trace"]
n = len(z["unnz"])
nt = (n + 31) // 32
t = buf[: 8 * nt].reshape(-1, 4)
base = t[0, 0]
t = t - base
ni = int(z["nitems"])
it = buf[8 * nt: 8 * nt + 4 * ni].reshape(-1, 4)
pe = it[:, 2] - base
row = (it[:, 3] & 0xffffffff) >> 3
cut = np.nonzero(np.diff(row) < -40)[0]
nl = int(cut[0]) + 1 if len(cut) else ni
slow_chain = (t[:, 2] - t[:, 1]) > 8000
late = []
for q in range(2 * nt):
    tile = q if q < nt else 2 * nt - 1 - q
    sel = slice(0, nl) if q < nt else slice(nl, ni)
    m = row[sel] // 32 == tile
    pub = pe[sel][m].max() if m.any() else -1
    late.append((t[q, 1] - t[q, 0]) > 8000 and pub < t[q, 0])
late = np.array(late)
print(f"{sys.argv[1]}: L {t[nt - 1, 2]} U {t[2 * nt - 1, 2] - t[nt - 1, 2]} cyc; slow chains "
      f"{slow_chain.sum()} ({(t[:, 2] - t[:, 1])[slow_chain].sum()} cyc), far-in stalls with "
      f"items ready {late.sum()} ({(t[:, 1] - t[:, 0])[late].sum()} cyc)")
