"""Per-stream timeline of one compress_batch + decompress step (CUDA events),
to separate device time from host-side gaps (plan readback -> encode launch)."""
import sys
import time

sys.path.insert(0, '/root/repo')
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import codec  # noqa: E402

torch.cuda.set_device(0)
ts, ebs, info, _ = bench.build_workload("alexnet256", "cuda")
ps = [pb.CodecParams(eb=e) for e in ebs]
outs = [torch.empty_like(t) for t in ts]
marks = []
orig_finish = codec._finish_compress


def traced_finish(x, p, dims, plan, dev, ctx, sh):
    s = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    h0 = time.perf_counter()
    r = orig_finish(x, p, dims, plan, dev, ctx, sh)
    h1 = time.perf_counter()
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(s)
    marks.append((x.numel(), e0, e1, h0, h1))
    return r


codec._finish_compress = traced_finish
for it in range(6):
    marks.clear()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    start.record()
    h_start = time.perf_counter()
    comp = pb.compress_batch(ts, ps)
    h_end = time.perf_counter()
    mid = torch.cuda.Event(enable_timing=True)
    mid.record()
    for (c, r), o in zip(comp, outs):
        pb.decompress_device(c, out=o, check=False)
    end = torch.cuda.Event(enable_timing=True)
    end.record()
    torch.cuda.synchronize()
    if it >= 4:
        print(f"step {it}: compress {start.elapsed_time(mid):.3f} ms, decompress {mid.elapsed_time(end):.3f} ms, "
              f"host in compress_batch {1e3 * (h_end - h_start):.3f} ms")
        for n, e0, e1, h0, h1 in marks:
            print(f"   n={n:9d} encode launched at {start.elapsed_time(e0):.3f} ms, encode done {start.elapsed_time(e1):.3f} ms,"
                  f" host finish() {1e3 * (h1 - h0):.3f} ms (host t={1e3 * (h0 - h_start):.3f})")
