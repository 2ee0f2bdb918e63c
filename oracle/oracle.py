"""ctypes wrapper of the CPU parity oracle (oracle/actc_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu-baseline legs of bench.py -- never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

OK, EPARAM, EDATA, EFORMAT, ENOMEM = 0, 1, 2, 3, 4


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "actc_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE, "-B", "liboracle.so"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P, U64, I64, D = C.c_void_p, C.c_uint64, C.c_int64, C.c_double
        L.orc_last_error.restype = C.c_char_p
        L.orc_prequantize_f64.argtypes = [P, U64, D, P]
        L.orc_prequantize_f32.argtypes = [P, U64, D, P]
        L.orc_lorenzo_encode.argtypes = [P, U64, U64, P, P]
        L.orc_lorenzo_encode.restype = U64
        L.orc_lorenzo_decode.argtypes = [P, U64, P, U64, U64, P]
        L.orc_build_code_lengths.argtypes = [P, U64, P]
        L.orc_canonical_codes.argtypes = [P, U64, P]
        L.orc_decode_bits.argtypes = [P, U64, U64, P, U64, P]
        L.orc_decode_bits.restype = I64
        L.orc_crc32.argtypes = [P, U64]
        L.orc_crc32.restype = C.c_uint32
        L.orc_compress.argtypes = [P, P, C.c_int, D, U64, C.c_int, C.POINTER(P)]
        for f in ("orc_result_n", "orc_result_k", "orc_result_blob_len", "orc_result_payload_bits", "orc_result_rle_runs"):
            getattr(L, f).argtypes = [P]
            getattr(L, f).restype = U64
        L.orc_result_copy.argtypes = [P, P, P, P, P]
        L.orc_free.argtypes = [P]
        L.orc_decompress_blob.argtypes = [P, U64, P, U64]
        L.orc_huffman_encode.argtypes = [P, U64, U64, P, P, P]
        L.orc_pairwise_sum_f32.argtypes = [P, U64]
        L.orc_pairwise_sum_f32.restype = C.c_float
        L.orc_pairwise_sum_f64.argtypes = [P, U64]
        L.orc_pairwise_sum_f64.restype = D
        for f in ("orc_mean_abs_f32", "orc_mean_abs_f64"):
            getattr(L, f).argtypes = [P, U64]
            getattr(L, f).restype = D
        for f in ("orc_count_nonzero_f32", "orc_count_nonzero_f64"):
            getattr(L, f).argtypes = [P, U64]
            getattr(L, f).restype = U64
        for f in ("orc_lbar_f32", "orc_lbar_f64"):
            getattr(L, f).argtypes = [P, U64, U64]
            getattr(L, f).restype = D
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _check(rc):
    if rc != OK:
        raise OracleError(rc, lib().orc_last_error().decode())


def prequantize(x, eb):
    x = np.ascontiguousarray(x)
    q = np.empty(x.size, dtype=np.int64)
    if x.dtype == np.float32:
        lib().orc_prequantize_f32(_p(x), x.size, float(eb), _p(q))
    else:
        x = np.ascontiguousarray(x, dtype=np.float64)
        lib().orc_prequantize_f64(_p(x), x.size, float(eb), _p(q))
    return q


def lorenzo_encode(lattice, radius, force=None):
    lat = np.ascontiguousarray(lattice, dtype=np.int64)
    sym = np.empty(lat.size, dtype=np.uint64)
    f = None if force is None else np.ascontiguousarray(force, dtype=np.uint8)
    lib().orc_lorenzo_encode(_p(lat), lat.size, int(radius), _p(f), _p(sym))
    return sym.astype(np.int64), np.flatnonzero(sym == 0).astype(np.int64)


def build_code_lengths(freqs):
    f = np.ascontiguousarray(freqs, dtype=np.uint64)
    out = np.empty(f.size, dtype=np.uint16)
    _check(lib().orc_build_code_lengths(_p(f), f.size, _p(out)))
    return out


def canonical_codes(lengths):
    l = np.ascontiguousarray(lengths, dtype=np.uint16)
    out = np.empty(l.size, dtype=np.uint64)
    lib().orc_canonical_codes(_p(l), l.size, _p(out))
    return out


def huffman_encode(symbols, alphabet):
    s = np.ascontiguousarray(symbols, dtype=np.uint64)
    lengths = np.empty(alphabet, dtype=np.uint16)
    payload = np.zeros(s.size * 8 + 16, dtype=np.uint8)
    bits = C.c_uint64(0)
    _check(lib().orc_huffman_encode(_p(s), s.size, int(alphabet), _p(lengths), _p(payload), C.byref(bits)))
    return lengths, payload[: (bits.value + 7) // 8].tobytes(), bits.value


def crc32(data: bytes) -> int:
    b = np.frombuffer(data, dtype=np.uint8)
    return int(lib().orc_crc32(_p(b), b.size))


class Compressed:
    """Result of the oracle compressor: blob + debug arrays."""

    def __init__(self, blob, symbols, hist, lengths, n, k, payload_bits, rle_runs):
        self.blob = blob
        self.symbols = symbols
        self.hist = hist
        self.lengths = lengths
        self.n = n
        self.k = k
        self.payload_bits = payload_bits
        self.rle_runs = rle_runs

    @property
    def ratio(self):
        return (self.n * 4) / len(self.blob)


def compress(x, eb, radius=1 << 15, preserve_zeros=True, debug=True):
    x = np.ascontiguousarray(x, dtype=np.float32)
    dims = np.asarray(x.shape if x.ndim else (1,), dtype=np.uint64)
    h = C.c_void_p()
    L = lib()
    _check(L.orc_compress(_p(x), _p(dims), int(dims.size), float(eb), int(radius), int(bool(preserve_zeros)), C.byref(h)))
    try:
        n = L.orc_result_n(h)
        blob = np.empty(L.orc_result_blob_len(h), dtype=np.uint8)
        sym = hist = lengths = None
        if debug:
            sym = np.empty(n, dtype=np.uint64)
            hist = np.empty(2 * radius, dtype=np.uint64)
            lengths = np.empty(2 * radius, dtype=np.uint16)
        L.orc_result_copy(h, _p(blob), _p(sym), _p(hist), _p(lengths))
        return Compressed(blob.tobytes(), sym, hist, lengths, n, L.orc_result_k(h),
                          L.orc_result_payload_bits(h), L.orc_result_rle_runs(h))
    finally:
        L.orc_free(h)


def decompress_blob(blob: bytes, n: int):
    b = np.frombuffer(blob, dtype=np.uint8)
    out = np.empty(max(n, 1), dtype=np.float64)
    _check(lib().orc_decompress_blob(_p(b), b.size, _p(out), n))
    return out[:n]


def pairwise_sum(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.float32:
        return np.float32(lib().orc_pairwise_sum_f32(_p(a), a.size))
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().orc_pairwise_sum_f64(_p(a), a.size)


def mean_abs(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.float32:
        return lib().orc_mean_abs_f32(_p(a), a.size)
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().orc_mean_abs_f64(_p(a), a.size)


def count_nonzero(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.float32:
        return int(lib().orc_count_nonzero_f32(_p(a), a.size))
    a = np.ascontiguousarray(a, dtype=np.float64)
    return int(lib().orc_count_nonzero_f64(_p(a), a.size))


def lbar(g):
    """training.py:360 -- mean over samples of max |g| per sample."""
    g = np.ascontiguousarray(g)
    N = g.shape[0]
    per = g.size // N
    if g.dtype == np.float32:
        return lib().orc_lbar_f32(_p(g), N, per)
    g = np.ascontiguousarray(g, dtype=np.float64)
    return lib().orc_lbar_f64(_p(g), N, per)


def inject_uniform_error(x, eb, preserve_zeros=True, seed=0):
    """errorprop.py:127-139 restated: numpy default_rng(seed) (PCG64) draws
    U[-eb, eb] noise for every element, zeroed where the input is 0 when
    preserve_zeros; returns f64(x) + noise (flat fp64)."""
    rng = np.random.default_rng(seed)
    data = np.asarray(x).astype(np.float64).reshape(-1)
    noise = rng.uniform(-eb, eb, size=data.size)
    if preserve_zeros:
        noise[data == 0.0] = 0.0
    return data + noise
