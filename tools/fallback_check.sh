timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_codebook.py tests/test_gpu_training.py -q -x -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do timeout 600 python bench.py --no-train --no-cpu --no-c1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['gpu_launches'], {k: round(v['busy_ms_per_step'],4) for k,v in d['kernels'].items()})"; done
timeout 600 python tools/redo_probe.py 2>&1 | grep -v Warn | tail -4
