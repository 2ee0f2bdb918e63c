"""Which stored activations of a torchvision model's compressed training need
the symbol-level fallback codebook (k2_codebook) instead of the frequency-
class kernel, and why (live symbols, classes, big-frequency symbols).
usage: python tools/fallback_probe.py resnet50 256"""
import os
import sys

os.environ["ACTC_K2_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torchvision  # noqa: E402

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import _lib, codec  # noqa: E402
from paper_2111_09562_b200.hooks import ActivationCompressor  # noqa: E402

name, batch = sys.argv[1], int(sys.argv[2])
dev = torch.device("cuda", 0)
torch.manual_seed(0)
m = getattr(torchvision.models, name)(num_classes=1000).to(dev)
opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
comp = ActivationCompressor(ActivationCompressor.conv_layer_map(m), opt, pb.ControllerConfig(W_default=2, W_floor=1))
x = torch.randn(batch, 3, 224, 224, device=dev)
y = torch.randint(0, 1000, (batch,), device=dev)
for i in range(6):
    if i == 4:
        comp.capture_next_iteration()
    opt.zero_grad(set_to_none=True)
    with comp.iteration():
        torch.nn.functional.cross_entropy(m(x), y).backward()
    opt.step()
    comp.after_step()
print("fallback shapes (n, radius):", sorted(codec._FALLBACK_SEEN))
L = _lib.lib()
L.actc_debug_k2_timing.argtypes = [C.c_void_p, C.c_void_p]
L.actc_debug_k2r_used.argtypes = [C.c_void_p]
for slot, (xh, c, eb) in comp.captured.items():
    t = torch.from_numpy(np.ascontiguousarray(xh)).to(dev)
    pb.compress_device(t, pb.CodecParams(eb=eb))
    used = L.actc_debug_k2r_used(_lib.context().handle)
    if not used:
        out = (C.c_uint64 * 32)()
        L.actc_debug_k2_timing(_lib.context().handle, out)
        v = list(out)
        why = {1: "L=0 / >2048 symbols with freq>=2^18 / sum>=2^32", 2: "classes > kRCap", 3: "phase caps (ni|nside, nph, R)",
               4: "code-length span / cut classes"}.get(v[20], "?")
        print(f"{slot}: n={t.numel()} eb={eb:.3g} -> fallback: {why}; vals {v[21]:#x} L={v[22]} {v[23]} {v[24]}")
