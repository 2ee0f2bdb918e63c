"""ctypes binding of the C ABI in include/actc.h (libactc.so, sm_100a).

The product path has no fallback: if the library is missing or no CUDA
device is present, every codec call raises.  PyTorch is used only for device
memory (caching allocator), streams and pinned host buffers.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DataError, FormatError, ParameterError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ACTC_LIB_PATH") or os.path.join(HERE, "libactc.so")  # override: A/B builds

ACTC_OK, ACTC_EPARAM, ACTC_EDATA, ACTC_EFORMAT, ACTC_ENOMEM, ACTC_ECUDA = range(6)
ACTC_FLAG_PRESERVE_ZEROS = 1
ACTC_ASYNC_K1_ONLY = 0x100
ACTC_ASYNC_REST = 0x200
ACTC_ASYNC_NO_FALLBACK = 0x400
ACTC_EAGAIN = 6
ACTC_TABLE_BYTES = 16400  # include/actc.h
ACTC_DEC_LUT_ONLY = 0x100
ACTC_DEC_REST = 0x200
ACTC_DEC_NO_NONZERO = 0x400
ACTC_DTYPE_F32, ACTC_DTYPE_F64 = 0, 1
ACTC_CHUNK = 128


class Plan(C.Structure):
    _fields_ = [
        ("n", C.c_uint64),
        ("n_outliers", C.c_uint64),
        ("payload_bits", C.c_uint64),
        ("live_symbols", C.c_uint32),
        ("max_len", C.c_uint32),
        ("rle_runs", C.c_uint64),
        ("entropy_bits", C.c_double),
        ("status", C.c_uint32),
        ("sym_bytes", C.c_uint32),
        ("sym_lo", C.c_uint32),
        ("sym_hi", C.c_uint32),
    ]


class StreamDesc(C.Structure):
    _fields_ = [
        ("n", C.c_uint64),
        ("eb", C.c_double),
        ("radius", C.c_uint32),
        ("flags", C.c_uint32),
        ("n_outliers", C.c_uint64),
        ("outlier_idx_dev", C.c_void_p),
        ("outlier_val_dev", C.c_void_p),
        ("live_symbols", C.c_uint32),
        ("canon_syms_dev", C.c_void_p),
        ("len_counts_dev", C.c_void_p),
        ("payload_dev", C.c_void_p),
        ("payload_bits", C.c_uint64),
        ("chunk_offsets_dev", C.c_void_p),
        ("chunk_lat_dev", C.c_void_p),
        ("table_dev", C.c_void_p),
    ]


class DecodeResult(C.Structure):
    _fields_ = [
        ("nonzero", C.c_uint64),
        ("markers", C.c_uint64),
        ("status", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


_lib = None
_lock = threading.Lock()


def lib():
    """Load libactc.so (raises if it is missing -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(make -C paper_2111_09562_b200/csrc)"
            )
        L = C.CDLL(LIB_PATH)
        P, U64, U32, D, I = C.c_void_p, C.c_uint64, C.c_uint32, C.c_double, C.c_int
        sig = {
            "actc_last_error": ([], C.c_char_p),
            "actc_version": ([], I),
            "actc_ctx_create": ([I, C.POINTER(P)], I),
            "actc_ctx_destroy": ([P], None),
            "actc_ctx_device_bytes": ([P], U64),
            "actc_ctx_take_status": ([P, P, P], I),
            "actc_debug_quant_check": ([D, U64, U64, P, P], I),
            "actc_ctx_set_scratch": ([P, P, U64], I),
            "actc_ctx_set_table_out": ([P, P, U64], I),
            "actc_compress_plan": ([P, P, U64, D, U32, U32, P, P, P], I),
            "actc_compress_encode": ([P, P, P, P, P, P, P, P, P, P], I),
            "actc_compress_async": ([P, P, U64, D, U32, U32, P, P, U64, P, P, U64, P, P, P, P, P], I),
            "actc_decompress": ([P, P, P, I, P, P], I),
            "actc_codebook_from_lengths": ([P, P, U64, P, P, P, P], I),
            "actc_build_chunk_index": ([P, P, P, P, P], I),
            "actc_crc32": ([P, P, U64, U32, P, P], I),
            "actc_memcpy_batch": ([P, P, P, I, P], I),
            "actc_inject_uniform": ([P, P, I, U64, D, I, P, P, P], I),
            "actc_prequantize": ([P, I, U64, D, P, P], I),
            "actc_lorenzo_encode": ([P, U64, U32, P, P, P, P], I),
            "actc_lorenzo_decode": ([P, U64, P, U64, U32, P, P, P], I),
            "actc_huffman_plan": ([P, P, U64, U64, P, P, P], I),
            "actc_huffman_encode": ([P, P, P, P, P, P, P, P], I),
            "actc_huffman_decode": ([P, P, P, P, P], I),
            "actc_code_lengths": ([P, P, U64, P, P, P], I),
            "actc_count_nonzero": ([P, I, U64, P, P], I),
            "actc_mean_abs": ([P, P, I, U64, P, P], I),
            "actc_lbar": ([P, P, I, U64, U64, P, P, P], I),
            "actc_timing_enable": ([I], I),
            "actc_kernel_stats": ([P, P, I], I),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


EXPORTED_SYMBOLS = (
    "actc_last_error actc_version actc_ctx_create actc_ctx_destroy actc_ctx_device_bytes actc_ctx_take_status actc_ctx_set_scratch actc_ctx_set_table_out actc_compress_plan "
    "actc_compress_encode actc_compress_async actc_decompress actc_codebook_from_lengths actc_build_chunk_index "
    "actc_prequantize actc_debug_quant_check actc_lorenzo_encode actc_lorenzo_decode actc_huffman_plan "
    "actc_huffman_encode actc_huffman_decode actc_code_lengths actc_count_nonzero "
    "actc_mean_abs actc_lbar actc_timing_enable actc_kernel_stats actc_crc32 actc_inject_uniform actc_memcpy_batch"
).split()

# instrumentation kinds (include/actc.h ACTC_KIND_*)
KERNEL_KINDS = ("quant", "codebook", "count", "scan", "pack", "fixup", "lut", "decode", "index", "stats", "debug", "crc", "inject")


def timing_enable(on: bool = True):
    """Bracket every library kernel launch with CUDA events on its stream."""
    lib().actc_timing_enable(1 if on else 0)


def kernel_stats() -> dict:
    """{kind: (launches, summed kernel ms)} since the last call; resets.
    Synchronizes the pending timing events."""
    n = len(KERNEL_KINDS)
    launches = (C.c_uint64 * n)()
    ms = (C.c_double * n)()
    raise_for(lib().actc_kernel_stats(C.cast(launches, C.c_void_p), C.cast(ms, C.c_void_p), n))
    return {k: (int(launches[i]), float(ms[i])) for i, k in enumerate(KERNEL_KINDS)}


def raise_for(rc: int, default_msg: str = ""):
    if rc == ACTC_OK:
        return
    msg = lib().actc_last_error().decode(errors="replace") or default_msg
    if rc == ACTC_EPARAM:
        raise ParameterError(msg)
    if rc == ACTC_EDATA:
        raise DataError(msg)
    if rc == ACTC_EFORMAT:
        raise FormatError(msg)
    if rc == ACTC_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA error in libactc: {msg}")


def cuda_available() -> bool:
    try:
        import torch
    except ImportError:
        return False
    return torch.cuda.is_available()


_TORCH_CUDA = None


def torch_cuda():
    """torch, once a CUDA device is known to be present (checked once per
    process: torch.cuda.is_available() re-reads the environment per call,
    and the codec's host path asks several times per compression)"""
    global _TORCH_CUDA
    if _TORCH_CUDA is not None:
        return _TORCH_CUDA
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2111_09562_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    _TORCH_CUDA = torch
    return torch


_tls = threading.local()


class Context:
    """One libactc context per (thread, device): owns device scratch."""

    def __init__(self, device: int):
        h = C.c_void_p()
        raise_for(lib().actc_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device
        torch = torch_cuda()
        # pinned host mailboxes for the async plan / decode-result copies
        self.plan_buf = torch.empty(C.sizeof(Plan), dtype=torch.uint8, pin_memory=True)
        self.dres_buf = torch.empty(C.sizeof(DecodeResult), dtype=torch.uint8, pin_memory=True)
        self.u64_buf = torch.empty(64, dtype=torch.uint8, pin_memory=True)
        self.sticky_buf = torch.zeros(4, dtype=torch.uint8, pin_memory=True)

    @property
    def plan(self) -> Plan:
        return Plan.from_address(self.plan_buf.data_ptr())

    @property
    def dres(self) -> DecodeResult:
        return DecodeResult.from_address(self.dres_buf.data_ptr())

    def __del__(self):
        try:
            lib().actc_ctx_destroy(self.handle)
        except Exception:
            pass


def context(device=None) -> Context:
    torch = torch_cuda()
    dev = torch.cuda.current_device() if device is None else int(device)
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    c = ctxs.get(dev)
    if c is None:
        with torch.cuda.device(dev):
            c = ctxs[dev] = Context(dev)
    return c


def release_contexts():
    """Destroy this thread's library contexts and their scratch (after a
    device synchronisation); they are recreated on next use."""
    torch = torch_cuda()
    torch.cuda.synchronize()
    for name in ("ctxs", "extra"):
        d = getattr(_tls, name, None)
        if d:
            d.clear()


def scratch_bytes(slots=None) -> int:
    """Device bytes held by this thread's library contexts (scratch the
    library cudaMalloc's itself, invisible to torch's allocator); `slots`
    restricts the sum to those context slots (0 = the main context)."""
    L = lib()
    ctxs = [(0, c) for c in getattr(_tls, "ctxs", {}).values()]
    ctxs += [(k[1], c) for k, c in getattr(_tls, "extra", {}).items()]
    return sum(int(L.actc_ctx_device_bytes(c.handle)) for sl, c in ctxs if slots is None or sl in slots)


def _thread_contexts(device):
    out = [c for d, c in getattr(_tls, "ctxs", {}).items() if d == device]
    out += [c for (d, _slot), c in getattr(_tls, "extra", {}).items() if d == device]
    return out


def take_decode_status(device=None, stream=None):
    """Queue the collection of every decode fault this thread's contexts on
    `device` saw since the last collection (actc_ctx_take_status) on
    `stream` (default: the device's current stream, which the batched
    decoders' side streams were joined into).  Returns an event; pass it to
    `decode_status_result` at the next natural synchronisation."""
    torch = torch_cuda()
    dev = torch.cuda.current_device() if device is None else int(device)
    sh, s = stream_handle(stream, dev)
    L = lib()
    for c in _thread_contexts(dev):
        raise_for(L.actc_ctx_take_status(c.handle, C.c_void_p(c.sticky_buf.data_ptr()), sh))
    return (dev, s.record_event())


def decode_status_result(token) -> int:
    """Wait for a take_decode_status event; ACTC_OK or ACTC_EFORMAT."""
    import torch

    dev, ev = token
    ev.synchronize()
    st = 0
    for c in _thread_contexts(dev):
        st |= int(c.sticky_buf.view(torch.int32).item())
        c.sticky_buf.zero_()
    return st


def context_for(device: int, slot: int) -> Context:
    """Extra contexts for concurrent (multi-stream) compression: slot 0 is
    the thread's main context, slots 1.. are private scratch sets."""
    if slot == 0:
        return context(device)
    torch = torch_cuda()
    extra = getattr(_tls, "extra", None)
    if extra is None:
        extra = _tls.extra = {}
    c = extra.get((device, slot))
    if c is None:
        with torch.cuda.device(device):
            c = extra[(device, slot)] = Context(device)
    return c


def current_stream():
    """torch.cuda.current_stream() of the current device without torch's
    per-call device-index resolution (which re-reads the environment: ~14 us
    a call, several per compression in training)."""
    torch = torch_cuda()
    sid, di, dt = torch._C._cuda_getCurrentStream(torch._C._cuda_getDevice())
    return torch.cuda.Stream(stream_id=sid, device_index=di, device_type=dt)


def stream_handle(stream=None, device=None):
    """(cudaStream_t handle, torch stream): `stream`, else the current stream
    of `device` (the tensor's device -- not necessarily the current one)."""
    torch = torch_cuda()
    s = torch.cuda.current_stream(device) if stream is None else stream
    return C.c_void_p(s.cuda_stream), s
