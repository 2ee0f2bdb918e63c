"""Host overhead of compress_begin / compress_end (small tensor, so the GPU
time is negligible): per-call microseconds and the cProfile top entries."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_09562_b200 import codec  # noqa: E402

x = torch.relu(torch.randn(64, 64, 32, 32, device="cuda"))
p = codec.CodecParams(eb=1e-3)
hint = None
for _ in range(20):
    j = codec.compress_begin([x], [p], slot_base=1, own_scratch=True)
    (c, r), = codec.compress_end(j, compact=True, order=False)
torch.cuda.synchronize()
N = 300
tb = te = 0.0
for _ in range(N):
    t0 = time.perf_counter()
    j = codec.compress_begin([x], [p], slot_base=1, own_scratch=True)
    t1 = time.perf_counter()
    j.jobs[0][2].synchronize()
    t2 = time.perf_counter()
    (c, r), = codec.compress_end(j, compact=True, order=False)
    t3 = time.perf_counter()
    tb += t1 - t0
    te += t3 - t2
print(f"compress_begin {1e6 * tb / N:.1f} us, compress_end (after the device finished) {1e6 * te / N:.1f} us per call")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    j = codec.compress_begin([x], [p], slot_base=1, own_scratch=True)
    (c, r), = codec.compress_end(j, compact=True, order=False)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
