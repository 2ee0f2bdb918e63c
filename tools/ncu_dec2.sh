#!/bin/bash
# ncu --set full of the decoder on bench layers 0 and 3; TAG
mkdir -p gpurun_out
for L in 0 3; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k4l_decode" -s 2 -c 1 \
   -o gpurun_out/${TAG}_dec$L -f python tools/prof_workload.py --steps 3 --only $L > gpurun_out/${TAG}_ncu$L.log 2>&1
ncu -i gpurun_out/${TAG}_dec$L.ncu-rep --page raw --csv > gpurun_out/${TAG}_dec${L}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_dec$L.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_dec${L}_src.csv 2>/dev/null
gzip -f gpurun_out/${TAG}_dec${L}_src.csv
done
