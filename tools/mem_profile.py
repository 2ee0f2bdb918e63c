"""Where the AlexNet b256 training peak sits: allocated bytes after the
forward pass and the max during backward, uncompressed vs compressed
(hooks, steady state)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torchvision  # noqa: E402

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200.hooks import ActivationCompressor  # noqa: E402

dev = torch.device("cuda")
for mode in ("baseline", "compressed"):
    torch.manual_seed(0)
    m = torchvision.models.alexnet(num_classes=1000).to(dev)
    opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
    comp = ActivationCompressor(ActivationCompressor.conv_layer_map(m), opt,
                                pb.ControllerConfig(W_default=2, W_floor=1)) if mode == "compressed" else None
    x = torch.randn(256, 3, 224, 224, device=dev)
    y = torch.randint(0, 1000, (256,), device=dev)
    for it in range(6):
        opt.zero_grad(set_to_none=True)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        if comp:
            with comp.iteration():
                loss = torch.nn.functional.cross_entropy(m(x), y)
                torch.cuda.synchronize()
                fwd = torch.cuda.memory_allocated()
                fwd_peak = torch.cuda.max_memory_allocated()
                torch.cuda.reset_peak_memory_stats()
                loss.backward()
        else:
            loss = torch.nn.functional.cross_entropy(m(x), y)
            torch.cuda.synchronize()
            fwd = torch.cuda.memory_allocated()
            fwd_peak = torch.cuda.max_memory_allocated()
            torch.cuda.reset_peak_memory_stats()
            loss.backward()
        torch.cuda.synchronize()
        bwd_peak = torch.cuda.max_memory_allocated()
        opt.step()
        if comp:
            comp.after_step()
        if it >= 4:
            print(f"{mode:10s} it{it}: start {base / 1e9:.3f} GB, after forward {fwd / 1e9:.3f}, forward peak {fwd_peak / 1e9:.3f}, backward peak {bwd_peak / 1e9:.3f}")
