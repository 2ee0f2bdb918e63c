"""Per-kind DRAM traffic and duration from an ncu capture of one bench step.

  ncu --set full -o gpurun_out/step python tools/prof_workload.py --steps 2
  ncu -i gpurun_out/step.ncu-rep --page raw --csv > gpurun_out/step_raw.csv
  python tools/ncu_traffic.py gpurun_out/step_raw.csv alexnet256 [launches_in_last_step]

Writes profiles/ncu_traffic.json[workload][kind] = dram bytes (read + write)
per launch, averaged over the last step's launches, and prints a summary.
bench.py reports it as roofline.traffic for the dominant kernel.
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KIND = {"k1_quant_lorenzo_hist": "quant", "k2_codebook": "codebook", "k2r_codebook": "codebook", "k2s_emit": "codebook",
        "k3_count": "count", "k3_seg_count": "count", "k_excl_scan_u64": "scan", "k3_cta_scan": "scan",
        "k3_pack": "pack", "k3_seg_pack": "pack", "k3_fixup": "fixup", "k_build_lut": "lut", "k_build_lut8": "lut",
        "k4w_decode": "decode", "k4x_decode": "decode", "k4_decode": "decode", "k4l_decode": "decode"}


def kernel_base(name):
    return name.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]


def load_raw(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    units = rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        d = {"name": kernel_base(r[h.index("Kernel Name")])}
        for m in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"):
            if m in h:
                i = h.index(m)
                v = float(r[i].replace(",", "") or 0)
                u = units[i]
                scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                         "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1.0)
                d[m] = v * scale
        out.append(d)
    return out


def main():
    path, workload = sys.argv[1], sys.argv[2]
    launches = load_raw(path)
    last = int(sys.argv[3]) if len(sys.argv) > 3 else len(launches)
    seq = launches[-last:]
    agg = collections.defaultdict(lambda: {"launches": 0, "us": 0.0, "dram": 0.0, "inst": 0.0})
    for d in seq:
        k = KIND.get(d["name"], d["name"])
        a = agg[k]
        a["launches"] += 1
        a["us"] += d.get("gpu__time_duration.sum", 0.0)
        a["dram"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a["inst"] += d.get("smsp__inst_executed.sum", 0.0)
    tot = sum(a["us"] for a in agg.values())
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        print(f"{k:10s} n={a['launches']:3d} {a['us']:9.1f}us ({100 * a['us'] / tot:4.1f}%) "
              f"dram/launch={a['dram'] / a['launches'] / 1e6:8.2f} MB  warp-inst={a['inst'] / 1e6:8.1f}M")
    dst = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    db = json.load(open(dst)) if os.path.exists(dst) else {}
    db[workload] = {k: a["dram"] / a["launches"] for k, a in agg.items()}
    db.setdefault("_about", "dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged over one "
                            "bench step captured with `ncu --set full --clock-control none` (tools/ncu_traffic.py)")
    with open(dst, "w") as fh:
        json.dump(db, fh, indent=1, sort_keys=True)
    print("wrote", dst)


if __name__ == "__main__":
    main()
