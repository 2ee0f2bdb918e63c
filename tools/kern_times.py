"""Per-kernel-kind device times of compress_device + decompress_device on
each bench tensor, run one tensor at a time (no overlap between tensors),
L2 flushed before each call: median over 7 reps, microseconds.
ACTC_LIB_PATH selects another build (A/B)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
ts, ebs, info, _, _ = bench.build_workload("alexnet256", "cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
for li, (t, eb) in enumerate(zip(ts, ebs)):
    p = pb.CodecParams(eb=eb)
    for _ in range(2):
        c, _ = pb.compress_device(t, p)
        pb.decompress_device(c, dtype=torch.float32)
    per = {}
    for _ in range(7):
        flush.zero_()
        torch.cuda.synchronize()
        _lib.timing_enable(True)
        c, _ = pb.compress_device(t, p)
        flush.zero_()
        pb.decompress_device(c, dtype=torch.float32, count_nonzero=False)
        torch.cuda.synchronize()
        _lib.timing_enable(False)
        rep = {}
        for kind, a, b in bench._timeline():
            rep[kind] = rep.get(kind, 0.0) + 1e3 * (b - a)
        for kind, v in rep.items():
            per.setdefault(kind, []).append(v)
    out[f"conv{li + 1}"] = {k: round(sorted(v)[len(v) // 2], 1) for k, v in per.items()}
tot = {}
for v in out.values():
    for k, x in v.items():
        tot[k] = round(tot.get(k, 0) + x, 1)
out["sum"] = tot
print(json.dumps(out))
