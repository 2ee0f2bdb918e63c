#!/bin/bash
# decoder micro-bench only (+ the decode parity tests); TAG=name
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_codec.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python tools/dec_bench.py > gpurun_out/${TAG}_dec.json 2>&1; tail -2 gpurun_out/${TAG}_dec.json
