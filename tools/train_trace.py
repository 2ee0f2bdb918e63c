"""torch.profiler trace of one compressed training iteration: kernel time per
stream and category, and the default stream's idle gaps.
usage: python tools/train_trace.py resnet50 256"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torchvision  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200.hooks import ActivationCompressor  # noqa: E402

name, batch = sys.argv[1], int(sys.argv[2])
dev = torch.device("cuda", 0)
torch.manual_seed(0)
m = getattr(torchvision.models, name)(num_classes=1000).to(dev)
opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
comp = ActivationCompressor(ActivationCompressor.conv_layer_map(m), opt, pb.ControllerConfig(W_default=2, W_floor=1))
x = torch.randn(batch, 3, 224, 224, device=dev)
y = torch.randint(0, 1000, (batch,), device=dev)


def it():
    opt.zero_grad(set_to_none=True)
    with comp.iteration():
        torch.nn.functional.cross_entropy(m(x), y).backward()
    opt.step()
    comp.after_step()


for _ in range(4):
    it()
comp.next_collection = comp.it + 1000
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    it()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0]
streams = collections.defaultdict(list)
for e in ev:
    streams[getattr(e, "device_resource_id", 0)].append(e)
t0 = min(e.time_range.start for e in ev)
t1 = max(e.time_range.end for e in ev)
print(f"iteration GPU span {(t1 - t0) / 1e3:.1f} ms")


def cat(nm):
    for k, c in (("k1_quant", "K1"), ("k2r", "K2r"), ("k2_codebook", "K2"), ("k2s_emit", "emit"), ("k3_seg_count", "count"),
                 ("k3_seg_pack", "pack"), ("k4l", "decode"), ("k4l_build", "table"), ("Memset", "memset"), ("Memcpy", "memcpy")):
        if k in nm:
            return c
    return "train"


for sid, es in sorted(streams.items(), key=lambda kv: -sum(e.time_range.elapsed_us() for e in kv[1])):
    tot = collections.Counter()
    for e in es:
        tot[cat(e.name)] += e.time_range.elapsed_us()
    es.sort(key=lambda e: e.time_range.start)
    busy = 0
    end = -1
    for e in es:
        s, f = e.time_range.start, e.time_range.end
        if s > end:
            busy += f - s
            end = f
        elif f > end:
            busy += f - end
            end = f
    print(f"stream {sid}: {len(es)} kernels, busy {busy / 1e3:.1f} ms of {(t1 - t0) / 1e3:.1f}; "
          + ", ".join(f"{k} {v / 1e3:.1f}" for k, v in tot.most_common()))

# the training stream's largest idle gaps: the kernels around them and what
# the other streams ran meanwhile
main_sid = max(streams, key=lambda k: sum(e.time_range.elapsed_us() for e in streams[k]))
es = sorted(streams[main_sid], key=lambda e: e.time_range.start)
gaps = []
for a, b in zip(es, es[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 50:
        gaps.append((g, a, b))
gaps.sort(key=lambda t: -t[0])
print(f"main stream gaps > 50 us: {len(gaps)}, total {sum(g for g, _, _ in gaps) / 1e3:.1f} ms")
for g, a, b in gaps[:12]:
    other = [e for sid, l in streams.items() if sid != main_sid for e in l
             if e.time_range.start < b.time_range.start and e.time_range.end > a.time_range.end]
    print(f"  {g / 1e3:.2f} ms at {(a.time_range.end - t0) / 1e3:.1f}: after {a.name[:40]!r} before {b.name[:40]!r}; "
          f"others: {collections.Counter(cat(e.name) for e in other).most_common(4)}")
