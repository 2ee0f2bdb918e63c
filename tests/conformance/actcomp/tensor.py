"""Tensor container and helpers: the drop-in's Tensor / make_tensor; the
reference's `compare` (error statistics of a reconstruction, tensor.py:195-216)
is test-harness arithmetic, restated here."""
from dataclasses import dataclass

import numpy as np

from paper_2111_09562_b200.errors import DimensionError, ParameterError
from paper_2111_09562_b200.tensor import Tensor, TensorStats, compute_stats, make_tensor  # noqa: F401


@dataclass(frozen=True)
class ErrorReport:
    eb: float
    max_abs_diff: float
    mean_abs_diff: float
    count_exceeding: int
    flushed_zero_count: int


def compare(a: Tensor, b: Tensor, eb: float) -> ErrorReport:
    if a.dims != b.dims:
        raise DimensionError(f"shape mismatch: {a.dims} vs {b.dims}")
    if eb < 0:
        raise ParameterError("eb must be >= 0")
    da = a.data.astype(np.float64)
    db = b.data.astype(np.float64)
    diff = np.abs(da - db)
    return ErrorReport(eb=float(eb), max_abs_diff=float(diff.max()), mean_abs_diff=float(diff.mean()),
                       count_exceeding=int(np.count_nonzero(diff > eb)),
                       flushed_zero_count=int(np.count_nonzero((db == 0.0) & (da != 0.0))))
