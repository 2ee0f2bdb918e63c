"""Host time per compressed training iteration spent in the hooks' codec
calls (compress_begin, compress_end split into device wait and the rest).
usage: python tools/host_cost.py resnet50 256"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torchvision  # noqa: E402

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import codec, hooks  # noqa: E402
from paper_2111_09562_b200.hooks import ActivationCompressor  # noqa: E402

acc = {"begin": 0.0, "end_total": 0.0, "end_wait": 0.0, "calls": 0}
_b, _e = codec.compress_begin, codec.compress_end
_sync = torch.cuda.Stream.synchronize


def begin(*a, **k):
    t = time.perf_counter()
    r = _b(*a, **k)
    acc["begin"] += time.perf_counter() - t
    acc["calls"] += 1
    return r


def sync(self):
    t = time.perf_counter()
    _sync(self)
    acc["end_wait"] += time.perf_counter() - t


def end(*a, **k):
    t = time.perf_counter()
    torch.cuda.Stream.synchronize = sync
    try:
        r = _e(*a, **k)
    finally:
        torch.cuda.Stream.synchronize = _sync
    acc["end_total"] += time.perf_counter() - t
    return r


hooks.compress_begin, hooks.compress_end = begin, end
name, batch = sys.argv[1], int(sys.argv[2])
dev = torch.device("cuda", 0)
torch.manual_seed(0)
m = getattr(torchvision.models, name)(num_classes=1000).to(dev)
opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
comp = ActivationCompressor(ActivationCompressor.conv_layer_map(m), opt, pb.ControllerConfig(W_default=2, W_floor=1))
x = torch.randn(batch, 3, 224, 224, device=dev)
y = torch.randint(0, 1000, (batch,), device=dev)
for i in range(8):
    if i == 4:
        comp.next_collection = comp.it + 1000
        for k in acc:
            acc[k] = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    opt.zero_grad(set_to_none=True)
    with comp.iteration():
        loss = torch.nn.functional.cross_entropy(m(x), y)
        tf = time.perf_counter()
        loss.backward()
    opt.step()
    comp.after_step()
    torch.cuda.synchronize()
    if i >= 4:
        print(f"iter {i}: wall {1e3 * (time.perf_counter() - t0):.1f} ms (forward host {1e3 * (tf - t0):.1f})", flush=True)
it = 4
print({k: (round(1e3 * v / it, 2) if k != "calls" else v // it) for k, v in acc.items()}, "ms per iteration")

if len(sys.argv) > 3:
    import cProfile
    import pstats

    pr = cProfile.Profile()
    for i in range(3):
        torch.cuda.synchronize()
        pr.enable()
        opt.zero_grad(set_to_none=True)
        with comp.iteration():
            torch.nn.functional.cross_entropy(m(x), y).backward()
        opt.step()
        comp.after_step()
        pr.disable()
    torch.cuda.synchronize()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(28)
