"""Device timeline of one bench step (compress_batch + decompress of the
alexnet256 activation set): every library launch with its stream slot and
start/end (ms, CUDA events), plus the step's host time."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import _lib  # noqa: E402

KIND = ["K1", "K2", "K3cnt", "scan", "K3pack", "fix", "lut", "K4dec", "idx", "stats", "dbg", "crc", "inject"]
torch.cuda.set_device(0)
ts, ebs, info, _ = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else "alexnet256", "cuda")
ps = [pb.CodecParams(eb=e) for e in ebs]
outs = [torch.empty_like(t) for t in ts]
L = _lib.lib()
L.actc_debug_timeline.argtypes = [C.POINTER(C.c_double), C.c_int]
L.actc_debug_timeline.restype = C.c_int
buf = (C.c_double * (4 * 4096))()
for it in range(5):
    torch.cuda.synchronize()
    L.actc_timing_enable(1 if it == 4 else 0)
    L.actc_debug_timeline(buf, 4096)
    h0 = time.perf_counter()
    comp = pb.compress_batch(ts, ps)
    h1 = time.perf_counter()
    pb.decompress_batch([c for c, _ in comp], outs)
    torch.cuda.synchronize()
    h2 = time.perf_counter()
L.actc_timing_enable(0)
n = L.actc_debug_timeline(buf, 4096)
print(f"host: compress_batch {1e3 * (h1 - h0):.3f} ms, total {1e3 * (h2 - h0):.3f} ms; {n} launches")
recs = sorted([(buf[4 * i + 1], buf[4 * i + 2], int(buf[4 * i]), int(buf[4 * i + 3])) for i in range(n)])
for t0, t1, k, sl in recs:
    print(f"  slot {sl}  {KIND[k]:7s} {t0:8.3f} -> {t1:8.3f}  ({1e3 * (t1 - t0):7.1f} us)")
