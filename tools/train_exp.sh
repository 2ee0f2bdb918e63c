for F in 8 2 1; do ACTC_FLUSH=$F python -c "
import sys, json; sys.argv=['bench.py']
import bench, torch
torch.cuda.set_device(0)
r = bench.run_training(None, 0, 1)
print('flush', $F, json.dumps({k: (v if k not in ('baseline','compressed') else {kk: vv for kk, vv in v.items() if kk != 'per_layer'}) for k, v in r.items()}))
"; done
