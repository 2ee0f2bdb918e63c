"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)")
ai, src = h.index("Address"), h.index("Source")
ex = h.index("Instructions Executed")
data = []
for i, r in enumerate(rows[2:]):
    try:
        data.append((float(r[si]), i, r[ai], r[src], r[ex]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
k = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for v, i, a, s, e in sorted(data, reverse=True)[:k]:
    print(f"{100 * v / tot:5.1f}%  #{i:5d} exec={e:>9} {s.strip()[:90]}")
