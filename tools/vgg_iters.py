"""Per-iteration times of the bench's VGG-16 compressed training leg (first
run in a fresh process): where does a slow first run spend its time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torchvision  # noqa: E402

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import codec  # noqa: E402
from paper_2111_09562_b200.hooks import ActivationCompressor  # noqa: E402

dev = torch.device("cuda", 0)
model = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
for rep, mode in enumerate(("baseline", "compressed", "baseline", "compressed")):
    torch.manual_seed(0)
    m = getattr(torchvision.models, model)(num_classes=1000).to(dev)
    opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
    comp = ActivationCompressor(ActivationCompressor.conv_layer_map(m), opt, pb.ControllerConfig(W_default=2, W_floor=1)) if mode == "compressed" else None
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(batch, 3, 224, 224, device=dev, generator=g)
    y = torch.randint(0, 1000, (batch,), device=dev, generator=g)
    for i in range(14):
        if i == 4 and comp:
            comp.next_collection = comp.it + 1000
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        opt.zero_grad(set_to_none=True)
        if comp:
            with comp.iteration():
                torch.nn.functional.cross_entropy(m(x), y).backward()
        else:
            torch.nn.functional.cross_entropy(m(x), y).backward()
        opt.step()
        if comp:
            comp.after_step()
        e1.record()
        e1.synchronize()
        st = torch.cuda.memory_stats(dev)
        print(rep, i, "gpu %.1f ms wall %.1f ms" % (e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)),
              "redos", len(codec.REDOS), "allocs", st["num_alloc_retries"], st["segment.all.allocated"],
              "reserved GB %.1f" % (st["reserved_bytes.all.current"] / 1e9), list(codec.REDOS)[-1:] if i in (7, 8) else "", flush=True)
