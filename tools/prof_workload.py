"""Run N compress+decompress steps of a bench workload (for ncu captures).

  ncu --set full -k regex:"k1_|k2_|k3_|k4_" -s 20 -c 4 -o prof python tools/prof_workload.py --steps 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2111_09562_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="alexnet256")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--only", type=int, default=-1, help="only this layer index")
args = ap.parse_args()
torch.cuda.set_device(0)
tensors, ebs, info, _, _ = bench.build_workload(args.workload, "cuda")
if args.only >= 0:
    tensors, ebs = [tensors[args.only]], [ebs[args.only]]
outs = [torch.empty_like(t) for t in tensors]
for _ in range(args.steps):
    for t, eb, o in zip(tensors, ebs, outs):
        c, rep = pb.compress_device(t, pb.CodecParams(eb=eb))
        pb.decompress_device(c, out=o, check=False, count_nonzero=False)
torch.cuda.synchronize()
print("done", [round(float(eb), 9) for eb in ebs])
