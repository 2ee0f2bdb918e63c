#!/bin/bash
# codec tests + decoder micro-bench + bench (no training legs); TAG=name
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_parity_large.py tests/test_gpu_internals.py tests/test_gpu_codebook.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/${TAG:-q}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG:-q}_pytest.log
tail -5 gpurun_out/${TAG:-q}_pytest.log
timeout 300 python tools/dec_bench.py > gpurun_out/${TAG:-q}_dec.json 2>&1; cat gpurun_out/${TAG:-q}_dec.json | tail -3
timeout 600 python bench.py --no-train --no-cpu > gpurun_out/${TAG:-q}_bench.json 2> gpurun_out/${TAG:-q}_bench.err; echo "bench rc=$?"
