#!/bin/bash
# codec tests (fast subset) + bench without training/cpu legs; TAG=name
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_internals.py tests/test_gpu_parity_large.py -q -x -p no:cacheprovider -k "not exhaustive and not 1gib and not payload_over" > gpurun_out/${TAG}_pytest.log 2>&1; tail -1 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --no-train --no-cpu > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench.json"))
print("value", round(d["value"],1), "ms", round(d["ms_per_step"],4), d["phase_ms_per_step"])
for k,v in d["kernels"].items(): print(k, {kk: (round(vv,4) if isinstance(vv,float) else vv) for kk,vv in v.items()})
print("c1", d.get("c1",{}).get("value"), d.get("c1",{}).get("phase_ms_per_step"))
PY
