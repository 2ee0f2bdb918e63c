#!/bin/bash
# codec parity tests + launch list of the bench steps; TAG=name
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_internals.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -2 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --no-train --no-cpu --no-c1 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]); print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],3), d['phase_ms_per_step'])"
TAG=${TAG} bash tools/gpu_launches.sh > /dev/null 2>&1; tail -25 gpurun_out/${TAG}_launch_summary.txt
