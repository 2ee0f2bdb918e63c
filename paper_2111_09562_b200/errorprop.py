"""Uniform error injection on the device (reference errorprop.py:127-139).

`inject_uniform_error(t, eb, preserve_zeros, seed)` adds i.i.d. U[-eb, +eb]
noise to every element (zeros keep zero noise when `preserve_zeros`) and
returns fp64, bit-identical to the reference: numpy's `default_rng(seed)`
is PCG64 seeded through SeedSequence; the host takes the generator state
numpy derives from the seed and K7 (`actc_inject_uniform`) replays the draws
on the device (LCG jump-ahead per thread, XSL-RR output, numpy's
`low + (high - low) * next_double`).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import ParameterError
from .tensor import Tensor

_M64 = (1 << 64) - 1


def _pcg64_state(seed) -> tuple[int, int]:
    st = np.random.PCG64(seed).state["state"]
    return int(st["state"]), int(st["inc"])


def inject_uniform_error(t, eb: float, preserve_zeros: bool = True, seed: int = 0):
    """Host `Tensor` in -> host fp64 `Tensor` out (the reference signature);
    a CUDA fp32/fp64 tensor in -> CUDA fp64 tensor out."""
    if not eb > 0:
        raise ParameterError(f"eb must be > 0, got {eb}")
    torch = _lib.torch_cuda()
    host = isinstance(t, Tensor)
    if host:
        x = torch.from_numpy(np.ascontiguousarray(t.data)).cuda()
    else:
        if not (t.is_cuda and t.dtype in (torch.float32, torch.float64)):
            raise ParameterError("inject_uniform_error expects a host Tensor or a CUDA fp32/fp64 tensor")
        x = t.contiguous()
    s, inc = _pcg64_state(seed)
    state = (C.c_uint64 * 4)(s >> 64, s & _M64, inc >> 64, inc & _M64)
    out = torch.empty(x.shape, dtype=torch.float64, device=x.device)
    sh, _ = _lib.stream_handle()
    dt = _lib.ACTC_DTYPE_F64 if x.dtype == torch.float64 else _lib.ACTC_DTYPE_F32
    _lib.raise_for(_lib.lib().actc_inject_uniform(_lib.context().handle, C.c_void_p(x.data_ptr()), dt, x.numel(),
                                                  float(eb), 1 if preserve_zeros else 0, C.cast(state, C.c_void_p),
                                                  C.c_void_p(out.data_ptr()), sh))
    if host:
        return Tensor(out.cpu().numpy().reshape(t.dims), precision=8)
    return out
