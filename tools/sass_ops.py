"""Executed warp-instructions by opcode (and hottest instructions) from an ncu sass source page csv."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ex, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot, cnt, lines = 0, {}, []
for i, r in enumerate(rows[2:]):
    try:
        e = float(r[ex])
    except (ValueError, IndexError):
        continue
    tot += e
    toks = r[src].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    cnt[op.split(".")[0]] = cnt.get(op.split(".")[0], 0) + e
    lines.append((e, i, r[src].strip()))
print("total warp-inst", tot)
print("  ".join(f"{k}:{100 * v / tot:.1f}%" for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:20]))
if len(sys.argv) > 2:
    lo, hi = int(sys.argv[2]), int(sys.argv[3])
    for e, i, s in lines:
        if lo <= i <= hi:
            print(f"#{i:5d} {e:12.0f} {s[:100]}")
