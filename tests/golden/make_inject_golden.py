"""Golden vectors for inject_uniform_error (reference errorprop.py:127-139),
produced by the reference itself in the build container.

It imports /root/reference/pkg/src/actcomp read-only and writes
tests/golden/inject_golden.npz: inputs (fp32 / fp64, with zeros), eb,
preserve flag, seed and the reference's fp64 output for each case.
"""
from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from actcomp import errorprop, tensor  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(2024)
    cases = []
    x = np.maximum(rng.normal(0, 1, (4, 8, 9, 9)), 0).astype(np.float32)  # ~50 % zeros
    cases.append((x, 1e-3, True, 0))
    cases.append((x, 1e-3, False, 7))
    cases.append((rng.normal(0, 3, 1000).astype(np.float64), 0.25, True, 123456789))
    cases.append((np.zeros(17, dtype=np.float32), 2.0, True, 5))
    cases.append((rng.uniform(-1, 1, 20001).astype(np.float32), 3.7e-6, True, 2 ** 40 + 3))
    out = {"numpy_version": np.array(np.__version__)}
    for i, (x, eb, pz, seed) in enumerate(cases):
        t = tensor.Tensor(x, precision=4 if x.dtype == np.float32 else 8)
        y = errorprop.inject_uniform_error(t, eb, preserve_zeros=pz, seed=seed)
        out[f"x_{i}"] = x
        out[f"y_{i}"] = np.asarray(y.data, dtype=np.float64)
        out[f"p_{i}"] = np.array([eb, float(pz), float(seed)])
    np.savez_compressed(os.path.join(HERE, "inject_golden.npz"), **out)
    print(f"{len(cases)} cases, numpy {np.__version__}")


if __name__ == "__main__":
    main()
