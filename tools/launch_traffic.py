"""Per-kind DRAM traffic per launch from an ncu launch list (tools/gpu_launches.sh:
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv),
averaged over the last `steps_launches` launches (default: one bench step, 25),
written to profiles/ncu_traffic.json[workload] -- bench.py's roofline.traffic.

  python tools/launch_traffic.py gpurun_out/r03_launches.csv alexnet256 25 r03
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KIND = {"k1_quant_lorenzo_hist": "quant", "k2r_codebook": "codebook", "k2_codebook": "codebook",
        "k2s_emit": "codebook", "k3_seg_count": "count", "k3_seg_pack": "pack", "k4l_decode": "decode",
        "k4_decode": "decode", "k4l_build_table": "lut", "k_build_lut": "lut"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
seq, order = {}, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = d["ID"]
    if k not in seq:
        seq[k] = {"name": d["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]}
        order.append(k)
    seq[k][d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
last = int(sys.argv[3]) if len(sys.argv) > 3 else 25
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for k in order[-last:]:
    d = seq[k]
    a = agg[KIND.get(d["name"], d["name"])]
    a[0] += 1
    a[1] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    a[2] += d.get("gpu__time_duration.sum", 0.0)
for kind, (nl, b, us) in sorted(agg.items(), key=lambda kv: -kv[1][2]):
    print(f"{kind:10s} launches {nl:3d}  {us:9.1f} us  dram/launch {b / nl / 1e6:8.2f} MB")
dst = os.path.join(ROOT, "profiles", "ncu_traffic.json")
db = json.load(open(dst)) if os.path.exists(dst) else {}
db[sys.argv[2]] = {kind: b / nl for kind, (nl, b, us) in agg.items()}
db["source"] = (f"ncu launch list of one bench step (profiles/{sys.argv[4] if len(sys.argv) > 4 else 'rNN'}_launches.csv): "
                "mean dram__bytes_read.sum + dram__bytes_write.sum per launch")
json.dump(db, open(dst, "w"), indent=1)
print("wrote", dst)
