"""bench.run_training for one model, repeated, with the decode prefetch on
and off (A/B in one process).  usage: python tools/leg_ab.py resnet50"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2111_09562_b200 import hooks  # noqa: E402

name = sys.argv[1]
orig = hooks.ActivationCompressor._prefetch_before
for rep in range(2):
    for pf in (True, False):
        hooks.ActivationCompressor._prefetch_before = orig if pf else (lambda self, h: None)
        leg = bench.run_training(name, bench.TRAIN_LEGS[name], 1)
        print(rep, "prefetch" if pf else "no-prefetch", round(leg["compressed"]["images_per_s"], 1),
              round(leg["baseline"]["images_per_s"], 1), flush=True)
