"""Markdown table of an ncu --set full capture (--page raw --csv): one row
per launch -- time, DRAM bytes and rate, warp instructions, occupancy,
issue activity and the three largest pc-sampled stall reasons."""
import csv
import sys


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
ix = {c: i for i, c in enumerate(h)}
units = rows[1]
TSCALE = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}
BSCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "KB": 1e-3, "MB": 1.0, "GB": 1e3}
t_scale = TSCALE.get(units[ix["gpu__time_duration.sum"]], 1.0)
stalls = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("_not_issued")]
print("| kernel | grid | time (us) | DRAM read+write (MB) | DRAM GB/s | warp-inst (M) | warps active % | issue active % | top stalls |")
print("|---|---|---|---|---|---|---|---|---|")
for r in rows[1:]:
    if len(r) != len(h) or not r[ix["Kernel Name"]] or r[ix["ID"]] in ("", "ID"):
        continue
    name = r[ix["Kernel Name"]].replace("void ", "").replace("actc::", "").split("(")[0]
    if not any(ch.isalpha() for ch in name):
        continue
    t = num(r[ix["gpu__time_duration.sum"]]) * t_scale  # us
    dram = (num(r[ix["dram__bytes_read.sum"]]) * BSCALE.get(units[ix["dram__bytes_read.sum"]], 1e-6)
            + num(r[ix["dram__bytes_write.sum"]]) * BSCALE.get(units[ix["dram__bytes_write.sum"]], 1e-6))  # MB
    inst = num(r[ix["smsp__inst_executed.sum"]]) / 1e6
    wa = num(r[ix["sm__warps_active.avg.pct_of_peak_sustained_active"]])
    ia = num(r[ix["smsp__issue_active.avg.pct_of_peak_sustained_active"]])
    s = sorted(((num(r[ix[c]]), c.replace("smsp__pcsamp_warps_issue_stalled_", "")) for c in stalls), reverse=True)
    tot = sum(v for v, _ in s) or 1.0
    top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in s[:3])
    print(f"| {name} | {r[ix['Grid Size']]} | {t:.1f} | {dram:.1f} | {dram * 1e3 / t if t else 0:.0f} | {inst:.1f} | {wa:.0f} | {ia:.0f} | {top} |")
