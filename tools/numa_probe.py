"""GPU-local CPU set (NVML) and pinned-copy bandwidth with and without
binding the process to it."""
import json
import os
import subprocess
import sys

import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
cpus = [64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
print("gpu-local cpus:", len(cpus), cpus[:8], "... of", os.cpu_count(), "current affinity", len(os.sched_getaffinity(0)))
here = os.path.dirname(os.path.abspath(__file__))
print("unbound:", subprocess.run([sys.executable, os.path.join(here, "pcie_bw.py")], capture_output=True, text=True).stdout.strip())
print("bound:  ", subprocess.run(["taskset", "-c", ",".join(map(str, cpus)), sys.executable, os.path.join(here, "pcie_bw.py")],
                                 capture_output=True, text=True).stdout.strip())
