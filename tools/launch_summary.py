"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ inst]): per kernel launch in order."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
seq = {}
order = []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    rec = dict(zip(hdr, r))
    key = rec['ID']
    if key not in seq:
        seq[key] = {'name': rec['Kernel Name'].split('(')[0].replace('void ', '')[:28], 'grid': rec['Grid Size']}
        order.append(key)
    v = float(rec['Metric Value'].replace(',', ''))
    seq[key][rec['Metric Name']] = v
last = int(sys.argv[2]) if len(sys.argv) > 2 else 60
for k in order[-last:]:
    d = seq[k]
    t = d.get('gpu__time_duration.sum', 0) / 1e3
    i = d.get('smsp__inst_executed.sum', 0)
    mb = (d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)) / 1e6
    gbs = mb / t * 1e-3 * 1e3 if t else 0.0
    print(f"{d['name']:28s} {d['grid']:>14s} {t:9.1f} us  inst {i:12.0f}  dram {mb:8.1f} MB {gbs:7.0f} GB/s")
