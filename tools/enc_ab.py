"""compress_device per tensor (CUDA events, median of 10, L2 flushed): the
bench workload's layers and C1."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2111_09562_b200 as pb
torch.cuda.set_device(0)
ts, ebs, info, _, _ = bench.build_workload("alexnet256", "cuda")
rng = np.random.default_rng(0)
c1 = torch.from_numpy(np.maximum(rng.normal(0, 1, (32, 64, 56, 56)), 0).astype(np.float32)).cuda()
ts = list(ts) + [c1]
ebs = list(ebs) + [1e-2 * float(c1.max() - c1.min())]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
for t, eb in zip(ts, ebs):
    p = pb.CodecParams(eb=eb)
    for _ in range(3):
        pb.compress_device(t, p)
    ms = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); pb.compress_device(t, p); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    res.append(round(1e3 * ms[5], 1))
print(json.dumps({"us": res}))
