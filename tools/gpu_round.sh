#!/bin/bash
# One GPU session: tests, bench, launch list, ncu --set full of one step.
# usage: tools/gpu_round.sh TAG [skip_tests]
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
if [ -z "$2" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  tail -3 gpurun_out/${TAG}_pytest.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2>> gpurun_out/${TAG}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k1_|k2|k3_|k_build|k4w_|k4x_|k4_" -c 400 --csv \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-train > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k1_|k2|k3_|k_build|k4w_|k4x_" -s 45 -c 45 \
   -o gpurun_out/${TAG}_step -f python tools/prof_workload.py --steps 2 > gpurun_out/${TAG}_ncu_full.log 2>&1
ncu -i gpurun_out/${TAG}_step.ncu-rep --page raw --csv > gpurun_out/${TAG}_step_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_step.ncu-rep --page details --csv > gpurun_out/${TAG}_step_details.csv 2>/dev/null
for k in k4w_decode k4x_decode k1_quant_lorenzo_hist k3_seg_pack k3_seg_count k2r_codebook; do
  ncu -i gpurun_out/${TAG}_step.ncu-rep --page source --csv --print-source sass -k regex:$k -c 1 > gpurun_out/${TAG}_src_$k.csv 2>/dev/null
done
# the copy-back limit is 64 MiB: keep the report only when small
sz=$(stat -c %s gpurun_out/${TAG}_step.ncu-rep 2>/dev/null || echo 0)
if [ "$sz" -gt 30000000 ]; then mv gpurun_out/${TAG}_step.ncu-rep /tmp/; fi
gzip -f gpurun_out/${TAG}_src_*.csv gpurun_out/${TAG}_step_raw.csv gpurun_out/${TAG}_step_details.csv
du -sh gpurun_out
ls -la gpurun_out | tail -20
