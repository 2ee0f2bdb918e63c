#!/bin/bash
# ncu --set full of K1 / count / pack on one bench tensor (compress_device path); TAG, LAYER
mkdir -p gpurun_out
L=${LAYER:-0}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_quant|k3_seg" -s 6 -c 3 \
   -o gpurun_out/${TAG}_enc -f python tools/prof_workload.py --steps 3 --only $L > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_enc.ncu-rep --page details --csv > gpurun_out/${TAG}_enc_details.csv 2>/dev/null
for k in k1_quant k3_seg_count k3_seg_pack; do
ncu -i gpurun_out/${TAG}_enc.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/${TAG}_src_$k.csv 2>/dev/null
done
tail -2 gpurun_out/${TAG}_ncu.log
