#!/bin/bash
# ncu --set full of the decoder on one bench tensor; TAG, LAYER (default 0)
mkdir -p gpurun_out
L=${LAYER:-0}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k4l_decode" -s 2 -c 1 \
   -o gpurun_out/${TAG}_dec -f python tools/prof_workload.py --steps 3 --only $L > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_dec.ncu-rep --page raw --csv > gpurun_out/${TAG}_dec_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_dec.ncu-rep --page details --csv > gpurun_out/${TAG}_dec_details.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_dec.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_dec_src.csv 2>/dev/null
tail -3 gpurun_out/${TAG}_ncu.log
