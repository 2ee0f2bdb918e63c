"""Timeline of bench.py's end-to-end step (pinned H2D -> compress ->
decompress -> D2H per tensor): CUDA-event timestamps per tensor, ms from
the step start."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2111_09562_b200 as pb  # noqa: E402

torch.cuda.set_device(0)
ts, ebs, info, _ = bench.build_workload("alexnet256", "cuda")
params = [pb.CodecParams(eb=e) for e in ebs]
host_in = [t.cpu().pin_memory() for t in ts]
host_out = [torch.empty(t.shape, dtype=torch.float32).pin_memory() for t in ts]
dev_in = [torch.empty_like(t) for t in ts]
outs = [torch.empty_like(t) for t in ts]
if os.environ.get("E2E_MAIN") == "side":
    torch.cuda.set_stream(torch.cuda.Stream())
stream = torch.cuda.current_stream()
print("main stream", stream, "legacy default" if stream.cuda_stream == 0 else "")
h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
order = sorted(range(len(ts)), key=lambda i: -ts[i].numel())
if len(sys.argv) > 1:
    order = [int(v) for v in sys.argv[1].split(",")]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


_orig_rec = torch.cuda.Stream.record_event


def _rec_timing(self, event=None):  # timing-capable events everywhere (the library's too)
    return _orig_rec(self, event if event is not None else torch.cuda.Event(enable_timing=True))


torch.cuda.Stream.record_event = _rec_timing


import time
from paper_2111_09562_b200 import codec as _pc

_HT = []
_ob, _oe = _pc.compress_begin, _pc.compress_end


def _tb(*a, **k):
    t = time.perf_counter()
    r = _ob(*a, **k)
    _HT.append(("begin", t, time.perf_counter()))
    return r


def _te(*a, **k):
    t = time.perf_counter()
    r = _oe(*a, **k)
    _HT.append(("end", t, time.perf_counter()))
    return r


_pc.compress_begin, _pc.compress_end = _tb, _te


def step(rec):
    _HT.clear()
    hs = time.perf_counter()
    hmarks = {}
    t0 = ev()
    t0.record(stream)
    h2d_s.wait_stream(stream)
    ready = {}
    for i in order:
        with torch.cuda.stream(h2d_s):
            dev_in[i].copy_(host_in[i], non_blocking=True)
        ready[i] = h2d_s.record_event(ev())
    marks = {}
    for i in order:
        ha = time.perf_counter()
        (c, _), = pb.compress_batch([dev_in[i]], [params[i]], ready=[ready[i]])
        hb = time.perf_counter()
        e_c = stream.record_event(ev())
        done = []
        pb.decompress_batch([c], [outs[i]], done=done)
        e_d = stream.record_event(ev())
        d2h_s.wait_event(done[0])
        if os.environ.get("E2E_D2H") == "raw":
            from cuda.bindings import runtime as rt
            err, = rt.cudaMemcpyAsync(host_out[i].data_ptr(), outs[i].data_ptr(), outs[i].numel() * 4,
                                      rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, d2h_s.cuda_stream)
        elif os.environ.get("E2E_NO_D2H") != "1":
            with torch.cuda.stream(d2h_s):
                host_out[i].copy_(outs[i], non_blocking=True)
        e_o = d2h_s.record_event(ev())
        hc = time.perf_counter()
        hmarks[i] = (1e3 * (ha - hs), 1e3 * (hb - hs), 1e3 * (hc - hs))
        marks[i] = (ready[i], e_c, e_d, e_o, done[0])
    stream.wait_stream(d2h_s)
    t1 = ev()
    t1.record(stream)
    rec.append((t0, t1, marks, hmarks, list(_HT), hs))


for _ in range(3):
    step([])
torch.cuda.synchronize()
import ctypes as C
from paper_2111_09562_b200 import _lib
L = _lib.lib()
L.actc_debug_timeline.argtypes = [C.POINTER(C.c_double), C.c_int]
L.actc_debug_timeline.restype = C.c_int
buf = (C.c_double * (4 * 4096))()
L.actc_debug_timeline(buf, 4096)
_lib.timing_enable(True)
rec = []
step(rec)
torch.cuda.synchronize()
_lib.timing_enable(False)
nrec = L.actc_debug_timeline(buf, 4096)
KIND = _lib.KERNEL_KINDS
recs = sorted((buf[4 * i + 1], buf[4 * i + 2], KIND[int(buf[4 * i])], int(buf[4 * i + 3])) for i in range(nrec))
t_first = recs[0][0] if recs else 0.0
t0, t1, marks, hmarks, ht, hs0 = rec[0]
print("host begin/end:", [(k, round(1e3 * (a - hs0), 2), round(1e3 * (b - hs0), 2)) for k, a, b in ht])
print(f"order {order}  total {t0.elapsed_time(t1):.2f} ms")
k1_t0 = None
for a, b, k, sl in recs:
    print(f"    kernel {k:9s} slot {sl}  {a:7.3f} -> {b:7.3f}")
for i in order:
    r, c, d, o, dd = marks[i]
    print(f"  t{i} {ts[i].numel() * 4 / 1e6:6.1f} MB  h2d done {t0.elapsed_time(r):6.2f}  compressed {t0.elapsed_time(c):6.2f}"
          f"  decoder done {t0.elapsed_time(dd):6.2f}  main after decode {t0.elapsed_time(d):6.2f}  d2h done {t0.elapsed_time(o):6.2f}"
          f"  | host: compress call {hmarks[i][0]:6.2f}-{hmarks[i][1]:6.2f}, d2h queued {hmarks[i][2]:6.2f}")
