#!/bin/bash
# round artifacts: full GPU test suite, bench (all legs), reference arm,
# launch list, ncu --set full of the decoder and encoder kernels; TAG=name
mkdir -p gpurun_out
T=${TAG:-final}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/${T}_smi.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
timeout 1500 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2>> gpurun_out/${T}_bench.err; echo "ref rc=$?"
TAG=${T} bash tools/gpu_launches.sh > /dev/null 2>&1
TAG=${T} bash tools/ncu_dec.sh > /dev/null 2>&1
TAG=${T} bash tools/ncu_enc.sh > /dev/null 2>&1
for f in gpurun_out/${T}_*.ncu-rep; do sz=$(stat -c %s $f); if [ "$sz" -gt 25000000 ]; then rm -f $f; fi; done
gzip -f gpurun_out/${T}_*src*.csv gpurun_out/${T}_dec_raw.csv 2>/dev/null
ls gpurun_out | grep ${T} | head -40
