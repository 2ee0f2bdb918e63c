"""Host-side profile of the bench step (compress_batch + decompress_batch)
under cProfile, plus the wall time from the end of the last compression
chain (its stream's synchronize returning) to the first decoder launch --
the stretch the GPU idles in between the two phases."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2111_09562_b200 import codec  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "alexnet256"
torch.cuda.set_device(0)
ts, ebs, info, _, _ = bench.build_workload(wl, "cuda")
ct = bench.CodecTimer(ts, ebs, "cuda")
for _ in range(5):
    ct.step()
torch.cuda.synchronize()

marks = {}
_sync = torch.cuda.Stream.synchronize


def sync(self):
    _sync(self)
    marks["last_sync"] = time.perf_counter()


torch.cuda.Stream.synchronize = sync
_dr = codec._decode_rest


def dr(*a):
    if "first_dec" not in marks:
        marks["first_dec"] = time.perf_counter()
    return _dr(*a)


codec._decode_rest = dr
from paper_2111_09562_b200 import _lib  # noqa: E402

_L = _lib.lib()
_ca = _L.actc_compress_async
calls = []


def ca(*a):
    r = _ca(*a)
    calls.append(time.perf_counter())
    return r


_L.actc_compress_async = ca
_cb, _db = codec.compress_batch, codec.decompress_batch
gaps = []
launch_t = []
for _ in range(30):
    ct.flush.zero_()
    torch.cuda.synchronize()
    marks.pop("first_dec", None)
    calls.clear()
    t0 = time.perf_counter()
    comp = ct.pb.compress_batch(ct.tensors, ct.params)
    t1 = time.perf_counter()
    launch_t.append([round((c - t0) * 1e6) for c in calls])
    ct.pb.decompress_batch([c for c, _ in comp], ct.outs)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    gaps.append(((t1 - marks["last_sync"]) * 1e6, (t2 - t1) * 1e6, (marks["first_dec"] - t1) * 1e6))
gaps.sort()
print("us from last stream sync to compress_batch return, decompress_batch host, return to first decoder call (median):", gaps[len(gaps) // 2])
print("us from compress_batch call to each actc_compress_async return (K1s, then the chains):", launch_t[len(launch_t) // 2])
torch.cuda.Stream.synchronize = _sync
pr = cProfile.Profile()
pr.enable()
for _ in range(30):
    ct.flush.zero_()
    ct.step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
