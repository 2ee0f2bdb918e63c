"""Timeline of one bench step of a workload (default c1): every GPU kernel
and memcpy with its start offset and duration relative to the step's first
GPU activity, from torch.profiler (CUPTI), plus the host-side time spent in
compress_batch / decompress_batch.  Shows where the step idles."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
torch.cuda.set_device(0)
if len(sys.argv) > 2:  # e.g. "alexnet256": run that workload's codec steps first (as bench.py does)
    ts0, ebs0, _, _, _ = bench.build_workload(sys.argv[2], "cuda")
    ct0 = bench.CodecTimer(ts0, ebs0, "cuda")
    ct0.timed(10)
    if len(sys.argv) > 3:
        ct0.step()
        del ts0, ct0
        torch.cuda.empty_cache()
ts, ebs, info, _, _ = bench.build_workload(wl, "cuda")
ct = bench.CodecTimer(ts, ebs, "cuda")
for _ in range(5):
    ct.step()
torch.cuda.synchronize()
hs = []
for _ in range(20):
    ct.flush.zero_()
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    comp = ct.pb.compress_batch(ct.tensors, ct.params)
    h1 = time.perf_counter()
    ct.pb.decompress_batch([c for c, _ in comp], ct.outs)
    h2 = time.perf_counter()
    torch.cuda.synchronize()
    hs.append(((h1 - h0) * 1e6, (h2 - h1) * 1e6))
hs.sort()
print("host us (compress_batch, decompress_batch), median:", hs[len(hs) // 2])
import gc
for mode in ("gc on", "gc off", "gc on"):
    if mode == "gc off":
        gc.collect()
        gc.disable()
    else:
        gc.enable()
    ms, ph = ct.timed(50)
    print(mode, "device step ms mean %.4f median %.4f" % (sum(ms) / len(ms), sorted(ms)[len(ms) // 2]),
          "sorted:", " ".join("%.3f" % v for v in sorted(ms)), "phases (sum):", ph)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        ct.flush.zero_()
        ct.step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
# last step: after the last flush kernel
idx = max(i for i, e in enumerate(evs) if e.time_range.end - e.time_range.start > 20 and
          ("fill" in e.name.lower() or "elementwise" in e.name.lower()))
t0 = evs[idx].time_range.end
for e in evs[idx + 1:]:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:90]}")
