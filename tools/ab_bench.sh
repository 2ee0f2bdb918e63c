#!/bin/bash
# codec parity subset on the in-tree build, then the bench step (no training,
# no CPU legs) on ab/libactc_*.so and the in-tree build, twice each; TAG=name
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_internals.py tests/test_gpu_parity_large.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -2 gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
for lib in ab/libactc_*.so in-tree; do
  if [ "$lib" = in-tree ]; then unset ACTC_LIB_PATH; else export ACTC_LIB_PATH=$lib; fi
  timeout 600 python bench.py --no-train --no-cpu --no-c1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', round(d['value'],1), round(d['ms_per_step'],4), {k: round(v['busy_ms_per_step'],4) for k,v in d['kernels'].items()})"
done; done
