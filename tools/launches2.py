"""Summarise an ncu launch list with gpu__time_duration.sum + smsp__inst_executed.sum per launch."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "")})
    d[r[mi]] = float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1)
last = int(sys.argv[2]) if len(sys.argv) > 2 else 45
seq = list(per.values())[-last:]
agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
for d in seq:
    a = agg[d["name"].split("<")[0]]
    a[0] += d.get("gpu__time_duration.sum", 0)
    a[1] += d.get("smsp__inst_executed.sum", 0)
    a[2] += 1
tot = sum(a[0] for a in agg.values())
for k, (t, inst, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:28s} n={c:2d} {t:9.1f}us ({100 * t / tot:4.1f}%)  warp-inst={inst / 1e6:8.1f}M")
print(" | ".join(f"{d['name'].split('<')[0]} {d.get('gpu__time_duration.sum', 0):.0f}" for d in seq))
