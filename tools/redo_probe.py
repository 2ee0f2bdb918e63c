import os, sys
sys.path.insert(0, "/root/repo")
import torch, torchvision
import paper_2111_09562_b200 as pb
from paper_2111_09562_b200 import codec
from paper_2111_09562_b200.hooks import ActivationCompressor
dev = torch.device("cuda", 0)
torch.manual_seed(0)
m = torchvision.models.resnet50(num_classes=1000).to(dev)
opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
comp = ActivationCompressor(ActivationCompressor.conv_layer_map(m), opt, pb.ControllerConfig(W_default=2, W_floor=1))
x = torch.randn(256, 3, 224, 224, device=dev); y = torch.randint(0, 1000, (256,), device=dev)
for i in range(16):
    if i == 4: comp.next_collection = comp.it + 1000
    n0 = len(codec.REDOS)
    opt.zero_grad(set_to_none=True)
    with comp.iteration():
        torch.nn.functional.cross_entropy(m(x), y).backward()
    opt.step(); comp.after_step()
    torch.cuda.synchronize()
    new = list(codec.REDOS)[n0:]
    if new: print(i, [(n, st, ml, no, kc, pbits, cb, round(pbits / max(cb, 1), 3)) for n, st, ml, no, kc, pbits, cb in new], flush=True)
print("done")
