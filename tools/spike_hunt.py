"""Hunt occasional slow training iterations: per-iteration GPU/host time,
cudaMalloc calls, allocator retries, redos and Python GC pauses.
usage: python tools/spike_hunt.py vgg16 128 30"""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torchvision  # noqa: E402

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import codec  # noqa: E402
from paper_2111_09562_b200.hooks import ActivationCompressor  # noqa: E402

name, batch, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda", 0)
gcs = []
_t = {}


def _gc_cb(phase, info):
    if phase == "start":
        _t["s"] = time.perf_counter()
    else:
        gcs.append((info["generation"], 1e3 * (time.perf_counter() - _t["s"])))


gc.callbacks.append(_gc_cb)
torch.manual_seed(0)
m = getattr(torchvision.models, name)(num_classes=1000).to(dev)
opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
comp = ActivationCompressor(ActivationCompressor.conv_layer_map(m), opt, pb.ControllerConfig(W_default=2, W_floor=1))
x = torch.randn(batch, 3, 224, 224, device=dev)
y = torch.randint(0, 1000, (batch,), device=dev)
for i in range(4 + iters):
    if i == 4:
        comp.next_collection = comp.it + 1000
    torch.cuda.synchronize()
    st0 = torch.cuda.memory_stats(dev)
    r0, g0 = len(codec.REDOS), len(gcs)
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    opt.zero_grad(set_to_none=True)
    with comp.iteration():
        torch.nn.functional.cross_entropy(m(x), y).backward()
    opt.step()
    comp.after_step()
    e1.record()
    th = 1e3 * (time.perf_counter() - t0)
    e1.synchronize()
    st1 = torch.cuda.memory_stats(dev)
    print(i, f"gpu {e0.elapsed_time(e1):.1f} host {th:.1f} ms", "malloc", st1.get("num_device_alloc", 0) - st0.get("num_device_alloc", 0),
          "retries", st1["num_alloc_retries"] - st0["num_alloc_retries"], "redos", len(codec.REDOS) - r0,
          "gc", [(g, round(d, 1)) for g, d in gcs[g0:] if d > 1], flush=True)
