"""Where a compressed training iteration's time goes: plain, hooks only
(first interval: stored activations raw, cheap layers recomputed), hooks +
codec.  usage: python tools/train_overhead.py resnet50 256"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torchvision  # noqa: E402

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200.hooks import ActivationCompressor  # noqa: E402

name, batch = sys.argv[1], int(sys.argv[2])
dev = torch.device("cuda", 0)
for mode in sys.argv[3].split(",") if len(sys.argv) > 3 else ("plain", "hooks_raw", "hooks_codec", "hooks_codec_inorder"):
    torch.manual_seed(0)
    m = getattr(torchvision.models, name)(num_classes=1000).to(dev)
    opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
    from paper_2111_09562_b200 import codec as _codec
    _codec._side_streams.clear()
    if "_pri0" in mode:  # side streams at the training stream's priority
        _codec._side_streams[0] = [torch.cuda.Stream(device=dev, priority=0) for _ in range(16)]
    comp = None
    if mode != "plain":
        w = 1000 if mode == "hooks_raw" else 2
        comp = ActivationCompressor(ActivationCompressor.conv_layer_map(m), opt,
                                    pb.ControllerConfig(W_default=w, W_floor=1),
                                    codec_on_compute_stream=mode.endswith("inorder"),
                                    prefetch_decode=not mode.endswith("nopf"),
                                    **({"batch_flush": int(mode.split("_bf")[1].split("_")[0])} if "_bf" in mode else {}))
    x = torch.randn(batch, 3, 224, 224, device=dev)
    y = torch.randint(0, 1000, (batch,), device=dev)

    def it():
        opt.zero_grad(set_to_none=True)
        if comp:
            with comp.iteration():
                torch.nn.functional.cross_entropy(m(x), y).backward()
        else:
            torch.nn.functional.cross_entropy(m(x), y).backward()
        opt.step()
        if comp:
            comp.after_step()

    for _ in range(4):
        it()
    if comp:
        comp.next_collection = comp.it + 1000
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    st0 = torch.cuda.memory_stats(dev)
    r0 = len(_codec.REDOS)
    evs[0].record()
    for i in range(6):
        it()
        evs[i + 1].record()
    evs[-1].synchronize()
    ms = evs[0].elapsed_time(evs[-1]) / 6
    st1 = torch.cuda.memory_stats(dev)
    per = [round(evs[i].elapsed_time(evs[i + 1]), 1) for i in range(6)]
    print(f"   per-iteration ms {per}; cudaMalloc calls {st1.get('num_device_alloc', 0) - st0.get('num_device_alloc', 0)}, "
          f"redos {len(_codec.REDOS) - r0}", flush=True)
    print(f"{name} b{batch} {mode}: {batch / ms * 1e3:.0f} img/s, {ms:.1f} ms/iter, "
          f"peak {torch.cuda.max_memory_allocated(dev) / 1e9:.2f} GB", flush=True)
    if comp:
        comp.remove()
    del m, opt, comp
    torch.cuda.empty_cache()
