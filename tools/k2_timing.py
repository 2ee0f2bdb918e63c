"""Per-stage K2 timing (clock64 cycles) for the bench workload's tensors:
frequency-class kernel (k2r) stages, or k2_codebook stages on fallback."""
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
tensors, ebs, info, _, _ = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else "alexnet256", "cuda")
L = _lib.lib()
L.actc_debug_k2_timing.argtypes = [C.c_void_p, C.c_void_p]
L.actc_debug_k2r_used.argtypes = [C.c_void_p]
for rep in range(2):
    for t, eb in zip(tensors, ebs):
        pb.compress_device(t, pb.CodecParams(eb=eb))
        used = L.actc_debug_k2r_used(_lib.context().handle)
        out = (C.c_uint64 * 32)()
        L.actc_debug_k2_timing(_lib.context().handle, out)
        v = list(out)
        if not rep:
            continue
        if used:
            st = ["classes", "class_ids", "phases", "levels", "per_class", "symbols", "plan"]
            d = {st[i]: v[i + 1] - v[i] for i in range(7)}
            print(f"k2r L={v[9]} classes={v[10]} iruns={v[11]} phases={v[8]} cut_classes={v[12]} "
                  f"total={v[7]-v[0]} cycles", d)
            if v[14] > v[5]:
                print("    symbols:", {"passA": (v[13] - v[5]) if v[13] > v[5] else 0, "prefixA": (v[14] - v[13]) if v[13] > v[5] else 0,
                                     "passB": v[15] - v[14], "prefixB": v[16] - v[15], "handover": v[6] - v[16]})
        else:
            st = ["compact", "sort", "phases", "depth", "canon", "plan"]
            d = {st[i]: v[i + 1] - v[i] for i in range(6) if v[i + 1] >= v[i]}
            print(f"k2 fallback L={v[9]} phases={v[8]} total={v[6]-v[0]} cycles", d)
