"""Decoder alone, one tensor at a time (CUDA events around actc_decompress on
the current stream, L2 flushed between reps): us per tensor and Gsym/s for
the bench workload's tensors.  ACTC_LIB_PATH selects an A/B build."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2111_09562_b200 as pb  # noqa: E402

torch.cuda.set_device(0)
ts, ebs, info, _, _ = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else "alexnet256", "cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
for t, eb in zip(ts, ebs):
    (c, rep), = pb.compress_batch([t], [pb.CodecParams(eb=eb)])
    out = torch.empty_like(t)
    for _ in range(3):
        pb.decompress_batch([c], [out])
    ms = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pb.decompress_batch([c], [out])
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    m = ms[len(ms) // 2]
    alg = rep.compressed_bytes + 4 * t.numel() + 16 * ((t.numel() + 127) // 128)
    res.append({"n": t.numel(), "live": c._live, "ratio": round(rep.ratio, 3), "us": round(1e3 * m, 1),
                "gsym_s": round(t.numel() / m / 1e6, 1), "alg_gbs": round(alg / m / 1e6, 1)})
print(json.dumps({"lib": os.environ.get("ACTC_LIB_PATH", "default"), 
                  "tensors": res, "total_us": round(sum(r["us"] for r in res), 1)}))
