timeout 900 python bench.py --no-cpu --no-c1 > gpurun_out/tr_all.json 2>/dev/null
timeout 900 python bench.py --no-cpu --no-c1 --train resnet50 > gpurun_out/tr_res.json 2>/dev/null
for f in tr_all tr_res; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
print('$f', d['value'], {m:(round(v['compressed']['images_per_s']), round(v['baseline']['images_per_s'])) for m,v in d['training'].items() if 'compressed' in v})"; done
