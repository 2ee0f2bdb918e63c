"""Per-SASS-line view of an ncu source page (--page source --csv
--print-source sass, gzipped): top stalled lines, shared/global wavefronts
per instruction, and totals per warp-level symbol step (argv[2] = symbols)."""
import csv
import gzip
import sys

rows = list(csv.reader(gzip.open(sys.argv[1], "rt")))[1:]
h = rows[0]
ix = {c: i for i, c in enumerate(h)}
rows = rows[1:]
steps = float(sys.argv[2]) / 32 if len(sys.argv) > 2 else 1.0


def g(x, c):
    try:
        return int(x[ix[c]] or 0)
    except (ValueError, KeyError):
        return 0


S, I = "Warp Stall Sampling (All Samples)", "Instructions Executed"
tot = sum(g(x, S) for x in rows)
ins = sum(g(x, I) for x in rows)
wf = sum(g(x, "L1 Wavefronts Shared") for x in rows)
print(f"samples {tot}  warp-inst {ins} ({ins / steps:.2f}/step)  shared wavefronts {wf} ({wf / steps:.2f}/step)")
for i in sorted(range(len(rows)), key=lambda i: -g(rows[i], S))[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    x = rows[i]
    print(f"{i:6d} {g(x, S):6d} {g(x, I):9d} {g(x, 'L1 Wavefronts Shared'):9d}  {x[ix['Source']].strip()[:80]}")
