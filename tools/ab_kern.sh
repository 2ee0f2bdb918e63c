#!/bin/bash
# codec parity subset on the in-tree build, then tools/kern_times.py on
# ab/libactc_*.so and the in-tree build; TAG=name
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_internals.py tests/test_gpu_parity_large.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
for lib in ab/libactc_*.so; do
  echo "$lib" >> gpurun_out/${TAG}_kern.json
  ACTC_LIB_PATH=$lib timeout 300 python tools/kern_times.py >> gpurun_out/${TAG}_kern.json 2>&1
done
echo "in-tree" >> gpurun_out/${TAG}_kern.json
timeout 300 python tools/kern_times.py >> gpurun_out/${TAG}_kern.json 2>&1
grep -v Warn gpurun_out/${TAG}_kern.json | tail -6
