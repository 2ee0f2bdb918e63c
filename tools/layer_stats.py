"""Per-layer alphabet statistics of the bench workload (diagnostic only):
live symbols L, distinct frequency values, max code length, bits/symbol and
the share of symbols whose codes exceed 12/14/16 bits."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2111_09562_b200 as pb  # noqa: E402

torch.cuda.set_device(0)
tensors, ebs, info, _ = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else "alexnet256", "cuda")
hists = []
for t, eb in zip(tensors, ebs):
    c, rep = pb.compress_device(t, pb.CodecParams(eb=eb))
    lens = c.code_lengths.astype(np.int64)
    x = t.reshape(-1).double()
    v = x / (2 * eb)
    q = torch.sign(v) * torch.floor(v.abs() + 0.5)
    d = torch.diff(q, prepend=torch.zeros(1, dtype=q.dtype, device=q.device)).long()
    r = 1 << 15
    d = torch.where(d.abs() < r, d + r, torch.zeros_like(d))
    h = torch.bincount(d, minlength=2 * r).cpu().numpy()
    live = h > 0
    hists.append(h)
    bits = (h * lens).sum()
    n = t.numel()
    share = {k: float(h[lens > k].sum() / n) for k in (10, 12, 14, 16, 20)}
    print(f"n={n} eb={eb:.3g} L={int(live.sum())} distinct_freqs={len(np.unique(h[live]))} "
          f"maxlen={int(lens.max())} bits/sym={bits / n:.3f} outliers={int(h[0])} share_gt={share} "
          f"ratio={rep.ratio:.3f}")
np.savez_compressed(os.path.join("gpurun_out", "layer_hists.npz"), *hists, ebs=np.array(ebs))
