"""Fraction of symbols the K4L decoder resolves off its 12-bit prefix table
(codes longer than the prefix, or prefixes shared by codes of two lengths),
per bench tensor, for prefix widths 12..14."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2111_09562_b200 as pb  # noqa: E402

ts, ebs, info, _, _ = bench.build_workload("alexnet256", "cuda")
for li, (t, eb) in enumerate(zip(ts, ebs)):
    c, rep = pb.compress_device(t, pb.CodecParams(eb=eb))
    lengths = c.code_lengths.astype(np.int64)
    # symbols: quantize + Lorenzo as the reference (fp64), outliers -> 0
    x = t.reshape(-1).double()
    q = torch.sign(x / (2 * eb)) * torch.floor(torch.abs(x / (2 * eb)) + 0.5)
    d = torch.diff(q, prepend=torch.zeros(1, dtype=q.dtype, device=q.device))
    R = c.params.radius
    sym = torch.where(d.abs() >= R, torch.zeros_like(d), d + R).long()
    freq = torch.bincount(sym, minlength=len(lengths)).cpu().numpy()
    n = freq.sum()
    L = lengths[np.arange(len(freq))]
    # canonical codes: (len, symbol) order
    live = np.nonzero(L)[0]
    order = live[np.lexsort((live, L[live]))]
    code = np.zeros(len(L), dtype=np.int64)
    cur, prev = 0, 0
    for s in order:
        cur <<= int(L[s]) - prev
        prev = int(L[s])
        code[s] = cur
        cur += 1
    out = []
    for k in (12, 13, 14):
        # a prefix resolves directly iff every code under it has one length <= k
        pre = {}
        for s in live:
            l = int(L[s])
            p = (code[s] << (k - l)) >> 0 if l <= k else code[s] >> (l - k)
            if l <= k:
                for pp in range(p, p + (1 << (k - l))):
                    pre.setdefault(pp, set()).add(l)
            else:
                pre.setdefault(p, set()).add(l)
        slow = 0
        for s in live:
            l = int(L[s])
            p = code[s] << (k - l) if l <= k else code[s] >> (l - k)
            if l > 31 or len(pre[p]) > 1:
                slow += freq[s]
        out.append(round(slow / n, 4))
    print(f"conv{li + 1}: live {len(live)} maxlen {L.max()} mixed-length prefixes (slow path) at 12/13/14 bits: {out}", flush=True)
