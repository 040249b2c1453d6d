"""Per-opcode and top-instruction warp-stall breakdown from an ncu source CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def f(r, h):
    try:
        return float(r[ix[h]] or 0)
    except (ValueError, IndexError):
        return 0.0


agg = collections.defaultdict(collections.Counter)
tot = 0.0
for r in data:
    toks = r[1].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
    for h in st:
        v = f(r, h)
        agg[op][h[6:]] += v
        tot += v
print("total samples", int(tot))
for t, op in sorted(((sum(c.values()), op) for op, c in agg.items()), reverse=True)[:14]:
    print(f"{op:14s} {t / tot:6.1%}", [(k, f"{v / tot:.1%}") for k, v in agg[op].most_common(3)])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("top instructions:")
for r in sorted(data, key=lambda r: -sum(f(r, h) for h in st))[:n]:
    s = sum(f(r, h) for h in st)
    top = sorted(((f(r, h), h[6:]) for h in st), reverse=True)[:2]
    print(f"{r[0][-5:]} {r[1][:58]:58s} {s / tot:5.1%} {[(k, int(v)) for v, k in top]}")
