#!/bin/bash
# decoder A/B: parity tests on the in-tree build, then tools/dec_bench.py on
# the in-tree build and on ab/libactc_*.so; TAG=name
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_internals.py tests/test_gpu_parity_large.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
for lib in ab/libactc_*.so; do
  ACTC_LIB_PATH=$lib timeout 300 python tools/dec_bench.py >> gpurun_out/${TAG}_dec.json 2>&1
done
timeout 300 python tools/dec_bench.py >> gpurun_out/${TAG}_dec.json 2>&1
cat gpurun_out/${TAG}_dec.json | tail -4
