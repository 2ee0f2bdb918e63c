#!/bin/bash
# tests + bench (+ reference arm) on one box.  usage: tools/r2_gpu.sh TAG [tests|bench|all]
TAG=${1:-r2}
WHAT=${2:-all}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
if [ "$WHAT" != "bench" ]; then
  timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  tail -3 gpurun_out/${TAG}_pytest.log
fi
if [ "$WHAT" != "tests" ]; then
  timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.json 2>> gpurun_out/${TAG}_bench.err; echo "ref rc=$?"
fi
