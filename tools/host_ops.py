"""Host cost (us, median of 200) of the individual operations compress_begin
performs per tensor, and of one whole compress_begin + compress_end for a
small tensor: where the ~50-80 us per launched chain go."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import _lib, codec  # noqa: E402


def med(f, k=200):
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return round(ts[k // 2] * 1e6, 2)


torch.cuda.set_device(0)
x = torch.randn(256, 64, 55, 55, device="cuda").relu_()
p = pb.CodecParams(eb=2e-4)
for _ in range(3):
    c, _ = pb.compress_batch([x], [p])[0]
torch.cuda.synchronize()
main = _lib.current_stream()
s = codec._stream_pool(0, 1)[0]
ctx = _lib.context_for(0, 1)
L = _lib.lib()
res = {
    "torch.empty(1 MB)": med(lambda: torch.empty(1 << 20, dtype=torch.uint8, device=x.device)),
    "_lib.current_stream": med(_lib.current_stream),
    "torch.cuda.current_stream": med(torch.cuda.current_stream),
    "_stream_pool": med(lambda: codec._stream_pool(0, 1)),
    "context_for": med(lambda: _lib.context_for(0, 1)),
    "record_event": med(main.record_event),
    "wait_event(record)": med(lambda: s.wait_event(main.record_event())),
    "record_stream": med(lambda: x.record_stream(s)),
    "x.is_contiguous + dtype": med(lambda: (x.is_contiguous(), x.dtype == torch.float32)),
    "x.data_ptr": med(x.data_ptr),
    "cudaMemsetAsync via torch zero_(8 B)": med(lambda: torch.zeros(1, dtype=torch.int64, device="cuda")),
    "ctx_set_table_out": med(lambda: L.actc_ctx_set_table_out(ctx.handle, 0, 0)),
}


def one():
    pend = codec.compress_begin([x], [p], slot_base=1)
    codec.compress_end(pend)


torch.cuda.synchronize()
res["compress_begin+end (conv1-size, incl. device time)"] = med(one, 50)


def begin_only():
    t0 = time.perf_counter()
    pend = codec.compress_begin([x], [p], slot_base=1)
    t1 = time.perf_counter()
    codec.compress_end(pend)
    return t1 - t0


ts = sorted(begin_only() for _ in range(50))
res["compress_begin alone"] = round(ts[25] * 1e6, 2)
for k, v in res.items():
    print(f"{v:9.2f}  {k}")
