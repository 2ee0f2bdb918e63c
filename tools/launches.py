"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[ui]]
        out.append((r[ki].split("(")[0].replace("void ", ""), v * scale))
    return out


if __name__ == "__main__":
    seq = load(sys.argv[1])
    last = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for n, us in seq[-last:]:
        tot[n] += us
        cnt[n] += 1
    print(f"last {last} launches (one timed step):")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"  {k:45s} n={cnt[k]:3d} total={v:9.1f}us avg={v / cnt[k]:8.1f}us")
    print("  sequence:", " | ".join(f"{n.split('<')[0]} {us:.0f}" for n, us in seq[-last:]))
