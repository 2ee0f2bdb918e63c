"""Canonical Huffman entry points (reference huffman.py), executed on the GPU.

build_code_lengths (huffman.py:37-75), canonical_codes (:78-94),
huffman_encode (:171-207) and huffman_decode (:210-236) call the same K2/K3/K4
kernels the codec uses; stream_entropy_bits (:239-246) is report arithmetic.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import FormatError, ParameterError
from .tensor import to_device

MAX_CODE_LENGTH = 63


def _u64_device(a):
    torch = _lib.torch_cuda()
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64).astype(np.uint64).view(np.int64))
    return torch.from_numpy(a).cuda()


def build_code_lengths(freqs) -> np.ndarray:
    torch = _lib.torch_cuda()
    f = np.asarray(freqs)
    A = len(f)
    if A == 0:
        return np.zeros(0, dtype=np.uint16)
    fd = _u64_device(f)
    lengths = torch.empty(A, dtype=torch.int16, device="cuda")
    ctx = _lib.context()
    sh, s = _lib.stream_handle()
    _lib.raise_for(_lib.lib().actc_code_lengths(ctx.handle, C.c_void_p(fd.data_ptr()), A, C.c_void_p(lengths.data_ptr()),
                                                 C.c_void_p(ctx.plan_buf.data_ptr()), sh))
    s.synchronize()
    if ctx.plan.status:
        raise ParameterError("Huffman code length exceeds 63 bits")
    return lengths.cpu().numpy().view(np.uint16)


def _canon_tables(lengths: np.ndarray):
    """device canonical table (canon symbols, per-length counts) from lengths"""
    torch = _lib.torch_cuda()
    A = len(lengths)
    live = int(np.count_nonzero(lengths))
    canon = torch.empty(max(live, 1), dtype=torch.int32, device="cuda")
    counts = torch.zeros(64, dtype=torch.int32, device="cuda")
    if live:
        dl = torch.from_numpy(np.ascontiguousarray(lengths.astype(np.uint16).view(np.int16))).cuda()
        ctx = _lib.context()
        sh, s = _lib.stream_handle()
        lh = C.c_uint32(0)
        _lib.raise_for(_lib.lib().actc_codebook_from_lengths(ctx.handle, C.c_void_p(dl.data_ptr()), A,
                                                              C.c_void_p(canon.data_ptr()), C.c_void_p(counts.data_ptr()),
                                                              C.byref(lh), sh))
    return canon, counts, live


def canonical_codes(lengths) -> np.ndarray:
    """Per-symbol canonical codes (uint64), 0 where length is 0."""
    lengths = np.asarray(lengths, dtype=np.int64)
    codes = np.zeros(len(lengths), dtype=np.uint64)
    if not np.any(lengths > 0):
        return codes
    canon, counts, live = _canon_tables(lengths.astype(np.uint16))
    canon_h = canon[:live].cpu().numpy().astype(np.int64)
    counts_h = counts.cpu().numpy().astype(np.int64)
    # first code per length (huffman.py:97-117 recurrence) + rank in canonical order
    first = np.zeros(64, dtype=object)
    code = 0
    for l in range(64):
        code <<= 1
        first[l] = code
        code += int(counts_h[l])
    base = np.concatenate(([0], np.cumsum(counts_h)[:-1]))
    lens_sorted = np.repeat(np.arange(64), counts_h)
    for i, (sym, l) in enumerate(zip(canon_h, lens_sorted)):
        codes[sym] = np.uint64(first[l] + (i - base[l]))
    return codes


def huffman_encode(symbols, alphabet_size: int):
    """Returns (lengths uint16[alphabet], payload bytes, bit_length)."""
    torch = _lib.torch_cuda()
    s_h = np.asarray(symbols, dtype=np.int64).reshape(-1)
    if alphabet_size < 1:
        raise ParameterError("alphabet_size must be >= 1")
    if s_h.size and (s_h.min() < 0 or s_h.max() >= alphabet_size):
        raise ParameterError("symbol out of alphabet range")
    n = s_h.size
    sym = to_device(np.ascontiguousarray(s_h.astype(np.uint32).view(np.int32))) if n else torch.zeros(1, dtype=torch.int32, device="cuda")
    lengths = torch.empty(alphabet_size, dtype=torch.int16, device="cuda")
    ctx = _lib.context()
    sh, s = _lib.stream_handle()
    L = _lib.lib()
    _lib.raise_for(L.actc_huffman_plan(ctx.handle, C.c_void_p(sym.data_ptr()), n, alphabet_size,
                                        C.c_void_p(lengths.data_ptr()), C.c_void_p(ctx.plan_buf.data_ptr()), sh))
    s.synchronize()
    plan = _lib.Plan.from_buffer_copy(ctx.plan)
    if plan.status:
        raise ParameterError("Huffman code length exceeds 63 bits")
    lens_h = lengths.cpu().numpy().view(np.uint16)
    if n == 0:
        return lens_h, b"", 0
    payload = torch.empty(4 * ((plan.payload_bits + 31) // 32) + 32, dtype=torch.uint8, device="cuda")
    canon = torch.empty(max(plan.live_symbols, 1), dtype=torch.int32, device="cuda")
    counts = torch.empty(64, dtype=torch.int32, device="cuda")
    chunk = torch.empty((n + _lib.ACTC_CHUNK - 1) // _lib.ACTC_CHUNK, dtype=torch.int64, device="cuda")
    _lib.raise_for(L.actc_huffman_encode(ctx.handle, C.c_void_p(sym.data_ptr()), C.byref(plan),
                                          C.c_void_p(payload.data_ptr()), C.c_void_p(canon.data_ptr()),
                                          C.c_void_p(counts.data_ptr()), C.c_void_p(chunk.data_ptr()), sh))
    nbytes = (plan.payload_bits + 7) // 8
    return lens_h, payload[:nbytes].cpu().numpy().tobytes(), int(plan.payload_bits)


def huffman_decode(lengths, payload: bytes, bit_length: int, count: int) -> np.ndarray:
    """Decode `count` symbols; FormatError on a malformed stream (huffman.py:210-236)."""
    torch = _lib.torch_cuda()
    if count == 0:
        return np.empty(0, dtype=np.int64)
    lengths = np.asarray(lengths, dtype=np.int64)
    if not np.any(lengths > 0):
        raise FormatError("empty code table with nonzero symbol count")
    if bit_length > len(payload) * 8:
        raise FormatError("payload shorter than declared bit length")
    if lengths.max() > MAX_CODE_LENGTH:
        raise FormatError("invalid code in bitstream")
    canon, counts, live = _canon_tables(lengths.astype(np.uint16))
    pb = np.zeros(4 * ((bit_length + 31) // 32) + 32, dtype=np.uint8)
    nbytes = (bit_length + 7) // 8
    pb[:nbytes] = np.frombuffer(payload, dtype=np.uint8)[:nbytes]
    pd = torch.from_numpy(pb).cuda()
    d = _lib.StreamDesc()
    d.n = count
    d.eb = 1.0
    d.radius = max(2, (len(lengths) + 1) // 2)
    d.flags = 0
    d.n_outliers = 0
    dummy = torch.zeros(2, dtype=torch.int64, device="cuda")
    d.outlier_idx_dev = dummy.data_ptr()
    d.outlier_val_dev = dummy.data_ptr()
    d.live_symbols = live
    d.canon_syms_dev = canon.data_ptr()
    d.len_counts_dev = counts.data_ptr()
    d.payload_dev = pd.data_ptr()
    d.payload_bits = bit_length
    d.chunk_offsets_dev = None
    d.chunk_lat_dev = None
    ctx = _lib.context()
    sh, s = _lib.stream_handle()
    nchunks = (count + _lib.ACTC_CHUNK - 1) // _lib.ACTC_CHUNK
    co = torch.zeros(nchunks, dtype=torch.int64, device="cuda")
    st = C.c_uint32(0)
    _lib.raise_for(_lib.lib().actc_build_chunk_index(ctx.handle, C.byref(d), C.c_void_p(co.data_ptr()), C.byref(st), sh))
    if st.value:
        raise FormatError("bitstream exhausted before all symbols decoded or invalid code")
    d.chunk_offsets_dev = co.data_ptr()
    out = torch.empty(count, dtype=torch.int32, device="cuda")
    _lib.raise_for(_lib.lib().actc_huffman_decode(ctx.handle, C.byref(d), C.c_void_p(out.data_ptr()),
                                                   C.c_void_p(ctx.dres_buf.data_ptr()), sh))
    s.synchronize()
    if ctx.dres.status:
        raise FormatError("invalid code in bitstream or bitstream length mismatch")
    return out.cpu().numpy().view(np.uint32).astype(np.int64)


def stream_entropy_bits(freqs) -> float:
    """Empirical Shannon entropy in bits/symbol (huffman.py:239-246)."""
    freqs = np.asarray(freqs, dtype=np.float64)
    total = freqs.sum()
    if total == 0:
        return 0.0
    p = freqs[freqs > 0] / total
    return float(-(p * np.log2(p)).sum())
