"""Host time inside compress_batch / decompress_batch, split by helper
(wrappers around the helpers; GPU work is not synchronised except where
compress_batch itself waits)."""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import _lib, codec  # noqa: E402

acc = collections.defaultdict(float)
cnt = collections.defaultdict(int)


def wrap(obj, name, label=None):
    f = getattr(obj, name)
    label = label or name

    def g(*a, **k):
        t0 = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            acc[label] += time.perf_counter() - t0
            cnt[label] += 1
    setattr(obj, name, g)


torch.cuda.set_device(0)
ts, ebs, info, _ = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else "alexnet256", "cuda")
ps = [pb.CodecParams(eb=e) for e in ebs]
outs = [torch.empty_like(t) for t in ts]
wrap(codec, "_container")
wrap(codec._DevBufs, "shrink")
wrap(codec._DevBufs, "carve")
wrap(codec.CompressedActivation, "_desc")
wrap(codec.CompressedActivation, "_record_stream")
wrap(torch.cuda.Stream, "synchronize", "stream.synchronize")
wrap(torch.cuda.Stream, "wait_event")
wrap(torch.cuda.Stream, "record_event")
wrap(_lib, "context_for")
L = _lib.lib()
for nm in ("actc_compress_async", "actc_decompress"):
    wrap(L, nm)
N = 30
for it in range(N + 5):
    if it == 5:
        acc.clear()
        cnt.clear()
        tc = td = 0.0
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    comp = pb.compress_batch(ts, ps)
    h1 = time.perf_counter()
    pb.decompress_batch([c for c, _ in comp], outs)
    h2 = time.perf_counter()
    torch.cuda.synchronize()
    if it >= 5:
        tc += h1 - h0
        td += h2 - h1
print(f"compress_batch host {1e6 * tc / N:.1f} us/call, decompress_batch host {1e6 * td / N:.1f} us/call")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:28s} {1e6 * v / N:8.1f} us/step  ({cnt[k] / N:.0f} calls)")
