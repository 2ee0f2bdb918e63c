"""Count the compress_end redos (synchronous re-compressions after a cap
overflow) of the bench's VGG-16 training leg and print its throughput."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2111_09562_b200 import codec  # noqa: E402

redos = []
_orig = codec.compress_device


def _wrap(x, p, *a, **k):
    redos.append((x.numel(), p.eb))
    return _orig(x, p, *a, **k)


codec.compress_device = _wrap
for r in range(3):
    leg = bench.run_training("vgg16", bench.TRAIN_LEGS["vgg16"], 1)
    print(r, round(leg["compressed"]["images_per_s"], 1), "redos so far", len(redos), len(codec.REDOS), flush=True)
