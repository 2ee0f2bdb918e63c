"""Per-stage K2 timing (clock64 cycles) for the bench workload's tensors."""
import ctypes as C
import os
import sys

os.environ["ACTC_K2_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
tensors, ebs, info, _ = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else "alexnet256", "cuda")
L = _lib.lib()
L.actc_debug_k2_timing.argtypes = [C.c_void_p, C.c_void_p]
for rep in range(2):
    for t, eb in zip(tensors, ebs):
        pb.compress_device(t, pb.CodecParams(eb=eb))
        out = (C.c_uint64 * 32)()
        L.actc_debug_k2_timing(_lib.context().handle, out)
        v = list(out)
        st = ["compact", "sort", "phases", "depth", "canon", "plan"]
        d = {st[i]: v[i + 1] - v[i] for i in range(6) if v[i + 1] >= v[i]}
        if rep:
            sub = {"init": v[10] - v[1], "pass0": v[11] - v[10], "pass1": v[12] - v[11], "pass2": v[13] - v[12],
                   "lb": v[16], "merge": v[17], "book": v[18]}
            print(f"L={v[9]} phases={v[8]} total={v[6]-v[0]} cycles", {k: int(x) for k, x in d.items()},
                  {k: int(x) for k, x in sub.items() if x < 1 << 40})
