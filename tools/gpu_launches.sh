#!/bin/bash
# launch list (ncu gpu__time_duration per kernel) of two bench steps; TAG=name
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k1_|k2|k3_|k_build|k4l_|k4_" -c 400 --csv \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-train --no-c1 > gpurun_out/${TAG}_under_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_summary.txt 2>&1; cat gpurun_out/${TAG}_launch_summary.txt | tail -30
