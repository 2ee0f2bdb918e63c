"""Tensor container and the activation statistics (GPU).

`Tensor` mirrors the reference's immutable host tensor
(/root/reference/pkg/src/actcomp/tensor.py:35-105): C-contiguous fp32/fp64,
NaN/Inf rejected at construction (DataError), read-only.  It is the drop-in
input/output type of compress/decompress; device-resident callers pass
torch CUDA tensors instead.

`compute_stats` (tensor.py:171-192) runs on the GPU through libactc: exact
nonzero count, numpy-order pairwise mean of |x|, exact maxima.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from .errors import DataError, DimensionError, ParameterError

_PRECISION_DTYPES = {4: np.float32, 8: np.float64}


def _validate_dims(dims: Sequence[int]) -> tuple[int, ...]:
    dims = tuple(int(d) for d in dims)
    if len(dims) == 0:
        raise DimensionError("tensor rank must be >= 1")
    if any(d < 1 for d in dims):
        raise DimensionError(f"all extents must be >= 1, got {dims}")
    if len(dims) > 255:
        raise DimensionError("rank exceeds 255")
    return dims


class Tensor:
    """Immutable dense tensor (reference tensor.py:35-105)."""

    __slots__ = ("_array",)

    def __init__(self, array, precision: int | None = None):
        arr = np.asarray(array)
        if precision is not None:
            if precision not in _PRECISION_DTYPES:
                raise ParameterError(f"precision must be 4 or 8, got {precision}")
            arr = arr.astype(_PRECISION_DTYPES[precision])
        elif arr.dtype != np.float32:
            arr = arr.astype(np.float64)
        _validate_dims(arr.shape)
        if not np.all(np.isfinite(arr)):
            raise DataError("tensor contains NaN or Inf")
        arr = np.ascontiguousarray(arr)
        arr.flags.writeable = False
        self._array = arr

    @property
    def dims(self) -> tuple[int, ...]:
        return self._array.shape

    @property
    def rank(self) -> int:
        return self._array.ndim

    @property
    def size(self) -> int:
        return self._array.size

    @property
    def precision(self) -> int:
        return self._array.dtype.itemsize

    @property
    def data(self) -> np.ndarray:
        return self._array.reshape(-1)

    def view(self) -> np.ndarray:
        return self._array

    def astype(self, precision: int) -> "Tensor":
        if precision == self.precision:
            return self
        return Tensor(self._array, precision=precision)

    def __eq__(self, other) -> bool:
        if not isinstance(other, Tensor):
            return NotImplemented
        return self.dims == other.dims and self.precision == other.precision and np.array_equal(self._array, other._array)

    def __hash__(self):
        return id(self)

    def __repr__(self) -> str:
        return f"Tensor(dims={self.dims}, precision={self.precision})"


@dataclass(frozen=True)
class TensorStats:
    nonzero_ratio: float
    mean_abs: float
    max_abs: float
    per_sample_max_abs: tuple[float, ...] = field(default_factory=tuple)


def make_tensor(dims, fill, *, value=0.0, lo=-1.0, hi=1.0, sparsity=0.5, seed=0, precision=8) -> Tensor:
    """Input generator with the reference's semantics (tensor.py:129-168)."""
    dims = _validate_dims(dims)
    n = int(np.prod(dims))
    if fill == "constant":
        flat = np.full(n, float(value), dtype=np.float64)
    elif fill == "uniform":
        if not hi >= lo:
            raise ParameterError(f"uniform fill needs hi >= lo, got [{lo}, {hi}]")
        flat = np.random.default_rng(seed).uniform(lo, hi, size=n)
    elif fill == "relu-sparse":
        if not 0.0 <= sparsity <= 1.0:
            raise ParameterError(f"sparsity must be in [0, 1], got {sparsity}")
        rng = np.random.default_rng(seed)
        flat = 1.0 - rng.random(n)
        zero_at = rng.permutation(n)[: int(round(sparsity * n))]
        flat[zero_at] = 0.0
    else:
        raise ParameterError(f"unknown fill spec {fill!r}")
    return Tensor(flat.reshape(dims), precision=precision)


# ---------------------------------------------------------------------------
# GPU statistics
# ---------------------------------------------------------------------------


def to_device(t, dtype=None):
    """Tensor / numpy / torch -> contiguous CUDA torch tensor (no copy if already)."""
    torch = _lib.torch_cuda()
    if isinstance(t, torch.Tensor):
        x = t
    else:
        arr = t.view() if isinstance(t, Tensor) else np.asarray(t)
        arr = np.ascontiguousarray(arr)
        x = torch.from_numpy(arr if arr.flags.writeable else arr.copy())
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    if not x.is_cuda:
        x = x.pin_memory().cuda(non_blocking=True) if x.numel() > (1 << 16) else x.cuda()
    return x.contiguous()


def _dtype_code(x):
    torch = _lib.torch_cuda()
    if x.dtype == torch.float32:
        return _lib.ACTC_DTYPE_F32
    if x.dtype == torch.float64:
        return _lib.ACTC_DTYPE_F64
    raise ParameterError(f"statistics need fp32/fp64 tensors, got {x.dtype}")


def count_nonzero(x, stream=None) -> int:
    """Exact nonzero count on the GPU (tensor.py:181)."""
    x = to_device(x)
    ctx = _lib.context(x.device.index)
    sh, s = _lib.stream_handle(stream, x.device)
    _lib.raise_for(_lib.lib().actc_count_nonzero(C.c_void_p(x.data_ptr()), _dtype_code(x), x.numel(),
                                                  C.c_void_p(ctx.u64_buf.data_ptr()), sh))
    s.synchronize()
    return int(ctx.u64_buf[:8].view(__import__("torch").int64).item())


def mean_abs(x, stream=None) -> float:
    """mean(|x|) with numpy's pairwise summation order, on the GPU."""
    x = to_device(x)
    ctx = _lib.context(x.device.index)
    sh, s = _lib.stream_handle(stream, x.device)
    _lib.raise_for(_lib.lib().actc_mean_abs(ctx.handle, C.c_void_p(x.data_ptr()), _dtype_code(x), x.numel(),
                                             C.c_void_p(ctx.u64_buf.data_ptr()), sh))
    s.synchronize()
    return float(ctx.u64_buf[:8].view(__import__("torch").float64).item())


def per_sample_max(x, stream=None):
    """(per-sample max |x| along axis 0 as a host tuple, mean of it the
    numpy way) -- training.py:360 / tensor.py:190-191."""
    torch = _lib.torch_cuda()
    x = to_device(x)
    ctx = _lib.context(x.device.index)
    sh, s = _lib.stream_handle(stream, x.device)
    N = x.shape[0] if x.dim() else 1
    out = torch.empty(N, dtype=x.dtype, device=x.device)
    _lib.raise_for(_lib.lib().actc_lbar(ctx.handle, C.c_void_p(x.data_ptr()), _dtype_code(x), N, x.numel() // N,
                                         C.c_void_p(out.data_ptr()), C.c_void_p(ctx.u64_buf.data_ptr()), sh))
    s.synchronize()
    lbar = float(ctx.u64_buf[:8].view(torch.float64).item())
    return tuple(float(v) for v in out.cpu().numpy()), lbar


def compute_stats(t, batch_dim: int | None = None) -> TensorStats:
    """GPU compute_stats (reference tensor.py:171-192)."""
    torch = _lib.torch_cuda()
    x = to_device(t)
    if x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float64)
    n = x.numel()
    nz = count_nonzero(x)
    mabs = mean_abs(x)
    per: tuple[float, ...] = ()
    flat_max, _ = per_sample_max(x.reshape(1, -1))
    max_abs = flat_max[0]
    if batch_dim is not None:
        if not 0 <= batch_dim < x.dim():
            raise DimensionError(f"batch_dim {batch_dim} out of range for rank {x.dim()}")
        moved = torch.movedim(x, batch_dim, 0).contiguous()
        per, _ = per_sample_max(moved)
    return TensorStats(nz / n, mabs, max_abs, per)
