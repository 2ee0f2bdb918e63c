"""Host-side cost of the library calls on the compress/decompress path (no sync inside the timed calls)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import _lib, codec  # noqa: E402

torch.cuda.set_device(0)
ts, ebs, info, _ = bench.build_workload("alexnet256", "cuda")
L = _lib.lib()
ctx = _lib.context()
sh, s = _lib.stream_handle()
t, eb = ts[0], ebs[0]
n = t.numel()
lat = torch.empty((n + 255) // 256, dtype=torch.int64, device="cuda")
for rep in range(3):
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    rc = L.actc_compress_plan(ctx.handle, C.c_void_p(t.data_ptr()), n, float(eb), 1 << 15, 1,
                              C.c_void_p(lat.data_ptr()), C.c_void_p(ctx.plan_buf.data_ptr()), sh)
    h1 = time.perf_counter()
    s.synchronize()
    plan = _lib.Plan.from_buffer_copy(ctx.plan)
    dev = codec._DevBufs()
    dev["chunk_lat"] = lat
    h2 = time.perf_counter()
    c, r = codec._finish_compress(t, pb.CodecParams(eb=eb), tuple(t.shape), plan, dev, ctx, sh)
    h3 = time.perf_counter()
    torch.cuda.synchronize()
    o = torch.empty_like(t)
    h4 = time.perf_counter()
    pb.decompress_batch([c], [o])
    h5 = time.perf_counter()
    torch.cuda.synchronize()
    h6 = time.perf_counter()
    pb.compress_batch(ts, [pb.CodecParams(eb=e) for e in ebs])
    h7 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"plan call {1e6*(h1-h0):.0f} us, finish (alloc+encode launches) {1e6*(h3-h2):.0f} us, "
          f"decompress_batch call {1e6*(h5-h4):.0f} us, compress_batch(5) host {1e6*(h7-h6):.0f} us")

# finer: the encode library call alone, and the Python around it
import cProfile
import pstats
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    pb.compress_batch(ts, [pb.CodecParams(eb=e) for e in ebs])
    pb.decompress_batch([c for c, _ in pb.compress_batch(ts, [pb.CodecParams(eb=e) for e in ebs])], [torch.empty_like(x) for x in ts])
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
