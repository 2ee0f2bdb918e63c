"""Drop-in codec API over the sm_100a kernels.

Mirrors /root/reference/pkg/src/actcomp/codec.py: `CodecParams` (:42-61),
`CompressionReport` (:64-71), `CompressedActivation` with the CMTZ byte
format (:74-179), `prequantize` (:238-251), `lorenzo_encode` (:254-272),
`lorenzo_decode` (:275-293), `compress` (:296-340), `decompress`
(:343-369), `write_compressed`/`read_compressed` (:372-386).

Every stage runs on the GPU through libactc (include/actc.h).  A
CompressedActivation produced by `compress` stays device-resident (payload,
outliers, canonical code table and the decode chunk index live in CUDA
memory); the reference's host fields (`payload`, `code_lengths`, ...) are
materialised lazily when accessed.  `decompress` returns the reference's fp64
host Tensor; `decompress_device` is the device path used by the training
hooks (fp32 output, no host round trip).
"""
from __future__ import annotations

import collections
import ctypes as C
import math
import struct
import warnings
import zlib
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import FormatError, ParameterError
from .tensor import Tensor, to_device

MAGIC_COMPRESSED = b"CMTZ"
COMPRESSED_FORMAT_VERSION = 1
PREDICTOR_IDS = {"lorenzo-1d": 1}
_PREDICTOR_NAMES = {v: k for k, v in PREDICTOR_IDS.items()}
_LATTICE_LIMIT = 1 << 61
DEFAULT_RADIUS = 1 << 15
_MAX_RUN = 0xFFFF


@dataclass(frozen=True)
class CodecParams:
    """User-facing knobs: absolute error bound and code alphabet size."""

    eb: float
    radius: int = DEFAULT_RADIUS
    predictor: str = "lorenzo-1d"
    preserve_zeros: bool = True

    def __post_init__(self):
        if not (self.eb > 0 and np.isfinite(self.eb)):
            raise ParameterError(f"eb must be a positive finite real, got {self.eb}")
        if self.radius < 2:
            raise ParameterError(f"radius must be >= 2, got {self.radius}")
        if self.predictor not in PREDICTOR_IDS:
            raise ParameterError(f"unknown predictor {self.predictor!r}")

    @property
    def alphabet_size(self) -> int:
        return 2 * self.radius


@dataclass(frozen=True)
class CompressionReport:
    original_bytes: int
    compressed_bytes: int
    ratio: float
    outlier_fraction: float
    codes_entropy_bits_per_symbol: float
    outlier_warning: bool


def _cmtz_size(rank: int, k: int, runs: int, bits: int) -> int:
    # header 53 + 8r, outliers 12k, RLE 4m, payload ceil(bits/8) (codec.py:95-119)
    return 53 + 8 * rank + 12 * k + 4 * runs + (bits + 7) // 8


def _rle_encode_lengths(lengths: np.ndarray) -> bytes:
    """codec.py:201-226 (host serialization helper)."""
    lengths = np.asarray(lengths, dtype=np.uint16)
    if lengths.size == 0:
        return struct.pack("<I", 0)
    change = np.flatnonzero(np.diff(lengths)) + 1
    starts = np.concatenate(([0], change))
    ends = np.concatenate((change, [lengths.size]))
    run_lens = ends - starts
    values = lengths[starts]
    if run_lens.max() > _MAX_RUN:
        reps = (run_lens + _MAX_RUN - 1) // _MAX_RUN
        vals = np.repeat(values, reps)
        lens = np.full(vals.size, _MAX_RUN, dtype=np.int64)
        last = np.cumsum(reps) - 1
        lens[last] = run_lens - (reps - 1) * _MAX_RUN
        run_lens, values = lens, vals
    runs = np.empty(len(run_lens), dtype=[("l", "<u2"), ("v", "<u2")])
    runs["l"] = run_lens
    runs["v"] = values
    return struct.pack("<I", len(run_lens)) + runs.tobytes()


class _Cursor:
    def __init__(self, buf: bytes):
        self.buf = buf
        self.pos = 0

    def take(self, n: int) -> bytes:
        if self.pos + n > len(self.buf):
            raise FormatError("truncated compressed stream")
        out = self.buf[self.pos : self.pos + n]
        self.pos += n
        return out

    def remaining(self) -> int:
        return len(self.buf) - self.pos


def _rle_decode_lengths(cur: _Cursor, alphabet_size: int) -> np.ndarray:
    (n_runs,) = struct.unpack("<I", cur.take(4))
    runs = np.frombuffer(cur.take(4 * n_runs), dtype=[("l", "<u2"), ("v", "<u2")])
    run_lens = runs["l"].astype(np.int64)
    if int(run_lens.sum()) != alphabet_size:
        raise FormatError("code-length table does not cover alphabet")
    return np.repeat(runs["v"], run_lens).astype(np.uint16)


def _payload_buffer_bytes(bits: int) -> int:
    # 4-byte words for the big-endian packer + 32 B over-read pad (the lane
    # decoder keeps six words of look-ahead)
    return 4 * ((bits + 31) // 32) + 32


class _DevBufs:
    """Device arrays of one container.  Arrays produced by the encoder are
    carved out of ONE uint8 allocation (`carve`); typed views are created
    only when a caller indexes them -- the hot path uses `ptr()`.  Arrays
    added individually (uploads, the lazily rebuilt index) are plain
    tensors.  Mapping-like: [], in, values(), ptr()."""

    __slots__ = ("_bufs", "_slots", "_views", "offsets")

    _DT = {"payload": "uint8", "out_idx": "int64", "out_val": "float32", "canon": "int32",
           "len_counts": "int32", "chunk_off": "int64", "chunk_lat": "int64"}

    def __init__(self):
        self._bufs = []      # backing tensors (carved bases and plain arrays)
        self._slots = {}     # name -> (base tensor, byte offset, numel, itemsize)
        self._views = {}
        self.offsets = {}

    def carve(self, device, layout):
        """layout: [(name, numel, itemsize)] -> one allocation, 16-byte aligned slots."""
        import torch

        offs, o = {}, 0
        for name, numel, isz in layout:
            offs[name] = o
            o += (numel * isz + 15) & ~15
        base = torch.empty(max(o, 16), dtype=torch.uint8, device=device)
        self._bufs.append(base)
        slots = self._slots
        for name, numel, isz in layout:
            slots[name] = (base, offs[name], numel, isz)
        self.offsets = offs
        return base

    def __setitem__(self, name, t):
        self._bufs.append(t)
        self._slots[name] = (t, 0, t.numel(), t.element_size())
        self._views[name] = t

    def __getitem__(self, name):
        v = self._views.get(name)
        if v is None:
            torch = _lib.torch_cuda()
            base, off, numel, isz = self._slots[name]
            v = base[off:off + numel * isz].view(getattr(torch, self._DT[name]))
            self._views[name] = v
        return v

    def __contains__(self, name):
        return name in self._slots

    def compact(self, names, stream, cur=None):
        """Move the named slots into one exact-size allocation (copies on
        `stream`); their old backing allocation is released once unused.
        `cur`: the caller's current stream (else looked up)."""
        torch = _lib.torch_cuda()
        olds = {self._slots[nm][0] for nm in names}
        layout = [(nm, self._slots[nm][2], self._slots[nm][3]) for nm in names]
        offs, o = {}, 0
        for nm, numel, isz in layout:
            offs[nm] = o
            o += (numel * isz + 15) & ~15
        if cur is None:
            cur = _lib.current_stream()
        # allocated on the caller's stream, read later there (the decoders);
        # a block the allocator hands out could still be in use by that
        # stream's queued work, so the copying stream waits for it first
        base = torch.empty(max(o, 16), dtype=torch.uint8, device=next(iter(olds)).device)
        if cur != stream:
            stream.wait_event(cur.record_event())
            base.record_stream(stream)
        # one library call queues every copy (torch slicing + copy_ per slot
        # costs ~10x the host time)
        k = len(layout)
        dst, src, nbs = (C.c_void_p * k)(), (C.c_void_p * k)(), (C.c_uint64 * k)()
        bp = base.data_ptr()
        for i, (nm, numel, isz) in enumerate(layout):
            sbase, soff, _, _ = self._slots[nm]
            dst[i], src[i], nbs[i] = bp + offs[nm], sbase.data_ptr() + soff, numel * isz
            self._slots[nm] = (base, offs[nm], numel, isz)
            self._views.pop(nm, None)
        _lib.raise_for(_lib.lib().actc_memcpy_batch(dst, src, nbs, k, C.c_void_p(stream.cuda_stream)))
        still = {self._slots[nm][0] for nm in self._slots}
        self._bufs = [b for b in self._bufs if b not in olds or b in still] + [base]

    def shrink(self, name, numel):
        """the slot's exact extent once the device plan is known (capped buffers)"""
        base, off, _, isz = self._slots[name]
        self._slots[name] = (base, off, int(numel), isz)
        self._views.pop(name, None)

    def ptr(self, name) -> int:
        base, off, _, _ = self._slots[name]
        return base.data_ptr() + off

    def values(self):
        return list(self._bufs)


class CompressedActivation:
    """Self-describing compressed container (reference codec.py:74-179).

    Constructed either from host fields (same signature as the reference's
    frozen dataclass) or, by `compress`, from device buffers.
    """

    __slots__ = (
        "dims", "precision", "params", "symbol_count", "payload_bits",
        "_h_outlier_indices", "_h_outlier_values", "_h_code_lengths", "_h_payload",
        "_dev", "_live", "_n_outliers", "_rle_runs", "_desc_cache", "_ready",
    )

    def __init__(self, dims, precision, params, outlier_indices, outlier_values, symbol_count,
                 code_lengths, payload, payload_bits):
        self.dims = tuple(int(d) for d in dims)
        self.precision = int(precision)
        self.params = params
        self.symbol_count = int(symbol_count)
        self.payload_bits = int(payload_bits)
        self._h_outlier_indices = np.asarray(outlier_indices, dtype=np.uint64)
        self._h_outlier_values = np.asarray(outlier_values, dtype=np.float32)
        self._h_code_lengths = np.asarray(code_lengths, dtype=np.uint16)
        self._h_payload = bytes(payload)
        self._dev = None
        self._live = None
        self._n_outliers = len(self._h_outlier_indices)
        self._rle_runs = None
        self._desc_cache = None
        self._ready = None

    # ---- device-resident construction (compress) ----
    @classmethod
    def _from_device(cls, dims, params, dev: dict, payload_bits: int, n_outliers: int, live: int, rle_runs: int):
        self = cls.__new__(cls)
        self.dims = tuple(int(d) for d in dims)
        self.precision = 4
        self.params = params
        n = 1
        for d in self.dims:
            n *= d
        self.symbol_count = n if self.dims else 0
        self.payload_bits = int(payload_bits)
        self._h_outlier_indices = None
        self._h_outlier_values = None
        self._h_code_lengths = None
        self._h_payload = None
        self._dev = dev
        self._live = int(live)
        self._n_outliers = int(n_outliers)
        self._rle_runs = int(rle_runs)
        self._desc_cache = None
        self._ready = None  # CUDA event: the device buffers are complete (compress_end(order=False))
        return self

    def _wait_ready(self, stream):
        """order `stream` after the work that fills the device buffers"""
        if self._ready is not None:
            stream.wait_event(self._ready)

    def _host_ready(self):
        """the device buffers are complete before a host read"""
        if self._ready is not None:
            self._ready.synchronize()

    @property
    def element_count(self) -> int:
        n = 1
        for d in self.dims:
            n *= d
        return n

    @property
    def is_device_resident(self) -> bool:
        return self._dev is not None

    @property
    def device(self):
        """CUDA device holding the container's buffers (uploaded to the
        current device on first use when built from host fields)."""
        return self._ensure_device()["payload"].device

    @property
    def device_nbytes(self) -> int:
        """Bytes held in device memory by this container (payload + side data)."""
        if self._dev is None:
            return 0
        return sum(t.numel() * t.element_size() for t in self._dev.values())

    # ---- reference host fields (materialised lazily) ----
    @property
    def outlier_indices(self) -> np.ndarray:
        self._host_ready()
        if self._h_outlier_indices is None:
            self._h_outlier_indices = self._dev["out_idx"].cpu().numpy().view(np.uint64).copy()
        return self._h_outlier_indices

    @property
    def outlier_values(self) -> np.ndarray:
        self._host_ready()
        if self._h_outlier_values is None:
            self._h_outlier_values = self._dev["out_val"].cpu().numpy().copy()
        return self._h_outlier_values

    @property
    def code_lengths(self) -> np.ndarray:
        self._host_ready()
        if self._h_code_lengths is None:
            canon = self._dev["canon"].cpu().numpy().astype(np.int64)
            counts = self._dev["len_counts"].cpu().numpy().astype(np.int64)
            lengths = np.zeros(self.params.alphabet_size, dtype=np.uint16)
            lengths[canon] = np.repeat(np.arange(64, dtype=np.uint16), counts)
            self._h_code_lengths = lengths
        return self._h_code_lengths

    @property
    def payload(self) -> bytes:
        self._host_ready()
        if self._h_payload is None:
            nbytes = (self.payload_bits + 7) // 8
            self._h_payload = self._dev["payload"][:nbytes].cpu().numpy().tobytes()
        return self._h_payload

    # ---- device upload (containers built from host fields) ----
    def _ensure_device(self):
        if self._dev is not None:
            return self._dev
        torch = _lib.torch_cuda()
        ctx = _lib.context()
        sh, s = _lib.stream_handle()
        dev = _DevBufs()
        nbytes = (self.payload_bits + 7) // 8
        if len(self._h_payload) < nbytes:
            raise FormatError("payload shorter than declared bit length")
        pb = np.zeros(_payload_buffer_bytes(self.payload_bits), dtype=np.uint8)
        pb[:nbytes] = np.frombuffer(self._h_payload, dtype=np.uint8)[:nbytes]
        dev["payload"] = torch.from_numpy(pb).cuda()
        dev["out_idx"] = torch.from_numpy(self._h_outlier_indices.view(np.int64).copy()).cuda()
        dev["out_val"] = torch.from_numpy(self._h_outlier_values.copy()).cuda()
        lengths = self._h_code_lengths
        A = self.params.alphabet_size
        if lengths.size != A:
            raise FormatError("code-length table does not cover alphabet")
        live = int(np.count_nonzero(lengths))
        dev["canon"] = torch.empty(max(live, 1), dtype=torch.int32, device="cuda")
        dev["len_counts"] = torch.zeros(64, dtype=torch.int32, device="cuda")
        if live:
            dl = torch.from_numpy(lengths.astype(np.uint16).view(np.int16).copy()).cuda()
            live_h = C.c_uint32(0)
            _lib.raise_for(_lib.lib().actc_codebook_from_lengths(
                ctx.handle, C.c_void_p(dl.data_ptr()), A, C.c_void_p(dev.ptr("canon")),
                C.c_void_p(dev.ptr("len_counts")), C.byref(live_h), sh))
        self._live = live
        self._dev = dev
        return dev

    def _record_stream(self, s):
        """mark the device buffers as in use on side stream s (caching allocator)"""
        if self._dev is not None:
            for t in self._dev.values():
                t.record_stream(s)

    def _desc(self, with_index=True) -> _lib.StreamDesc:
        if with_index and self._desc_cache is not None:
            return self._desc_cache
        dev = self._dev
        ptr = dev.ptr
        p = self.params
        # positional construction: one ctypes call instead of 15 attribute sets
        # (this runs per container between a batch's last compression and its
        # first decoder launch)
        d = _lib.StreamDesc(
            self.symbol_count, float(p.eb), int(p.radius),
            _lib.ACTC_FLAG_PRESERVE_ZEROS if p.preserve_zeros else 0, self._n_outliers,
            ptr("out_idx"), ptr("out_val"), self._live, ptr("canon"), ptr("len_counts"), ptr("payload"),
            self.payload_bits,
            ptr("chunk_off") if (with_index and "chunk_off" in dev) else None,
            ptr("chunk_lat") if (with_index and "chunk_lat" in dev) else None,
            ptr("table") if (with_index and "table" in dev) else None)
        if with_index and d.chunk_offsets_dev:
            self._desc_cache = d  # device buffers are fixed for the container's lifetime
        return d

    def _ensure_index(self):
        dev = self._ensure_device()
        if "chunk_off" in dev:
            return
        torch = _lib.torch_cuda()
        ctx = _lib.context()
        sh, s = _lib.stream_handle()
        n = self.symbol_count
        if n and not self._live:
            raise FormatError("empty code table with nonzero symbol count")
        nchunks = (n + _lib.ACTC_CHUNK - 1) // _lib.ACTC_CHUNK
        co = torch.zeros(max(nchunks, 1), dtype=torch.int64, device="cuda")
        st = C.c_uint32(0)
        d = self._desc(with_index=False)
        _lib.raise_for(_lib.lib().actc_build_chunk_index(ctx.handle, C.byref(d), C.c_void_p(co.data_ptr()),
                                                          C.byref(st), sh))
        if st.value:
            raise FormatError("bitstream does not decode to the declared symbol count")
        dev["chunk_off"] = co

    # ---- CMTZ (codec.py:95-179) ----
    def to_bytes(self) -> bytes:
        flags = 1 if self.params.preserve_zeros else 0
        head = MAGIC_COMPRESSED + struct.pack(
            "<Bd I BB", COMPRESSED_FORMAT_VERSION, self.params.eb, self.params.radius,
            PREDICTOR_IDS[self.params.predictor], flags,
        )
        head += struct.pack("<BB", self.precision, len(self.dims))
        head += struct.pack(f"<{len(self.dims)}Q", *self.dims)
        out = bytearray(head)
        idx = self.outlier_indices
        out += struct.pack("<Q", len(idx))
        if len(idx):
            pairs = np.empty(len(idx), dtype=[("i", "<u8"), ("v", "<f4")])
            pairs["i"] = idx
            pairs["v"] = self.outlier_values
            out += pairs.tobytes()
        out += struct.pack("<Q", self.symbol_count)
        out += _rle_encode_lengths(self.code_lengths)
        out += struct.pack("<Q", self.payload_bits)
        if self._dev is None:
            out += self.payload
            out += struct.pack("<I", zlib.crc32(out))
            return bytes(out)
        # device-resident payload: its CRC is taken on the device (K6,
        # continuing the host CRC of the prefix) and the payload is copied
        # once, straight into the blob
        nbytes = (self.payload_bits + 7) // 8
        pre = len(out)
        self._host_ready()
        crc = crc32_device(self._dev["payload"], nbytes, zlib.crc32(out))
        blob = bytearray(pre + nbytes + 4)
        blob[:pre] = out
        if nbytes:
            torch = _lib.torch_cuda()
            view = torch.frombuffer(blob, dtype=torch.uint8, count=nbytes, offset=pre)
            view.copy_(self._dev["payload"][:nbytes])
            del view
        blob[pre + nbytes:] = struct.pack("<I", crc)
        return bytes(blob)

    @classmethod
    def from_bytes(cls, blob: bytes) -> "CompressedActivation":
        if len(blob) < 4 + 1 + 8 + 4 + 2 + 2 + 4:
            raise FormatError("compressed stream too short")
        body, (stored_crc,) = blob[:-4], struct.unpack("<I", blob[-4:])
        if _body_crc(body) != stored_crc:
            raise FormatError("checksum mismatch")
        cur = _Cursor(body)
        if cur.take(4) != MAGIC_COMPRESSED:
            raise FormatError("bad magic")
        version, eb, radius, predictor_id, flags = struct.unpack("<Bd I BB", cur.take(15))
        if version != COMPRESSED_FORMAT_VERSION:
            raise FormatError(f"unsupported version {version}")
        if predictor_id not in _PREDICTOR_NAMES:
            raise FormatError(f"unknown predictor id {predictor_id}")
        try:
            params = CodecParams(eb=eb, radius=radius, predictor=_PREDICTOR_NAMES[predictor_id],
                                 preserve_zeros=bool(flags & 1))
        except ParameterError as exc:
            raise FormatError(f"invalid codec params in header: {exc}") from exc
        precision, rank = struct.unpack("<BB", cur.take(2))
        if rank == 0:
            raise FormatError("rank must be >= 1")
        dims = struct.unpack(f"<{rank}Q", cur.take(8 * rank))
        if any(d < 1 for d in dims):
            raise FormatError(f"bad extents {dims}")
        (n_out,) = struct.unpack("<Q", cur.take(8))
        if n_out:
            pairs = np.frombuffer(cur.take(12 * n_out), dtype=[("i", "<u8"), ("v", "<f4")])
            out_idx = pairs["i"].astype(np.uint64)
            out_val = pairs["v"].astype(np.float32)
        else:
            out_idx = np.empty(0, dtype=np.uint64)
            out_val = np.empty(0, dtype=np.float32)
        (symbol_count,) = struct.unpack("<Q", cur.take(8))
        lengths = _rle_decode_lengths(cur, 2 * radius)
        (payload_bits,) = struct.unpack("<Q", cur.take(8))
        payload = cur.take((payload_bits + 7) // 8)
        if cur.remaining():
            raise FormatError("trailing bytes in compressed stream")
        return cls(dims=tuple(int(d) for d in dims), precision=precision, params=params,
                   outlier_indices=out_idx, outlier_values=out_val, symbol_count=int(symbol_count),
                   code_lengths=lengths, payload=bytes(payload), payload_bits=int(payload_bits))

    def __repr__(self):
        return (f"CompressedActivation(dims={self.dims}, eb={self.params.eb}, bits={self.payload_bits}, "
                f"outliers={self._n_outliers}, device={self.is_device_resident})")


# ---------------------------------------------------------------------------
# compress / decompress
# ---------------------------------------------------------------------------


def compress_device(x, params: CodecParams, dims=None, stream=None):
    """Compress a contiguous fp32 CUDA tensor; returns (CompressedActivation, CompressionReport).

    One host synchronisation (the compressed size is data dependent); all
    buffers come from the torch caching allocator.
    """
    torch = _lib.torch_cuda()
    if x.dtype != torch.float32:
        raise ParameterError("compress expects a 32-bit tensor; convert explicitly with astype(4)")
    if not x.is_contiguous():
        x = x.contiguous()
    dims = tuple(x.shape) if dims is None else tuple(dims)
    if len(dims) == 0:
        dims = (1,)
    n = x.numel()
    ctx = _lib.context(x.device.index)
    sh, s = _lib.stream_handle(stream, x.device)
    L = _lib.lib()
    flags = _lib.ACTC_FLAG_PRESERVE_ZEROS if params.preserve_zeros else 0
    nchunks = (n + _lib.ACTC_CHUNK - 1) // _lib.ACTC_CHUNK
    chunk_lat = torch.empty(nchunks, dtype=torch.int64, device=x.device)
    _lib.raise_for(L.actc_compress_plan(ctx.handle, C.c_void_p(x.data_ptr()), n, float(params.eb),
                                        int(params.radius), flags, C.c_void_p(chunk_lat.data_ptr()),
                                        C.c_void_p(ctx.plan_buf.data_ptr()), sh))
    s.synchronize()
    plan = _lib.Plan.from_buffer_copy(ctx.plan)
    dev = _DevBufs()
    dev["chunk_lat"] = chunk_lat
    return _finish_compress(x, params, dims, plan, dev, ctx, sh)


def _check_plan(plan):
    if plan.status:
        if plan.status == _lib.ACTC_EDATA:
            from .errors import DataError
            raise DataError("tensor contains NaN or Inf")
        raise ParameterError("Huffman code length exceeds 63 bits")


def _finish_compress(x, params, dims, plan, dev, ctx, sh):
    """phase 2 (K3 encode) into exact-size buffers; returns (container, report)."""
    n = x.numel()
    _check_plan(plan)
    # one allocation per container, carved (the host cost per tensor is on
    # the critical path of compress_batch)
    k, live = plan.n_outliers, max(plan.live_symbols, 1)
    base = dev.carve(x.device, [("chunk_off", (n + _lib.ACTC_CHUNK - 1) // _lib.ACTC_CHUNK, 8),
                                ("out_idx", k, 8), ("payload", _payload_buffer_bytes(plan.payload_bits), 1),
                                ("out_val", k, 4), ("canon", live, 4), ("len_counts", 64, 4)])
    bp = base.data_ptr()
    o = dev.offsets
    rc = _lib.lib().actc_compress_encode(ctx.handle, x.data_ptr(), C.byref(plan), bp + o["payload"],
                                         bp + o["out_idx"], bp + o["out_val"], bp + o["canon"],
                                         bp + o["len_counts"], bp + o["chunk_off"], sh)
    if rc:
        _lib.raise_for(rc)
    return _container(n, params, dims, plan, dev)


def _container(n, params, dims, plan, dev):
    c = CompressedActivation._from_device(dims, params, dev, plan.payload_bits, plan.n_outliers,
                                          plan.live_symbols, plan.rle_runs)
    blob_len = _cmtz_size(len(dims), plan.n_outliers, plan.rle_runs, plan.payload_bits)
    frac = plan.n_outliers / n
    report = CompressionReport(
        original_bytes=n * 4, compressed_bytes=blob_len, ratio=(n * 4) / blob_len, outlier_fraction=frac,
        codes_entropy_bits_per_symbol=float(plan.entropy_bits), outlier_warning=frac > 0.5,
    )
    return c, report


def crc32_device(buf, nbytes: int, value: int = 0) -> int:
    """zlib.crc32(bytes(buf[:nbytes]), value) of a CUDA byte buffer (K6,
    actc_crc32) -- the CMTZ checksum (codec.py:118, :126).  Synchronizes."""
    torch = _lib.torch_cuda()
    if not buf.is_cuda or buf.element_size() * buf.numel() < nbytes or not buf.is_contiguous():
        raise ParameterError("crc32_device needs a contiguous CUDA buffer of at least nbytes bytes")
    out = C.c_uint32(0)
    sh, _ = _lib.stream_handle()
    _lib.raise_for(_lib.lib().actc_crc32(_lib.context().handle, C.c_void_p(buf.data_ptr()), int(nbytes),
                                         int(value) & 0xFFFFFFFF, C.byref(out), sh))
    del torch
    return int(out.value)


_DEVICE_CRC_MIN = 4 << 20  # blobs from disk: below this, zlib on the host is as fast as the upload


def _body_crc(body) -> int:
    """CRC of a host blob body: on the device for large blobs when a GPU is
    present (upload + K6 beats zlib's ~2.5 GB/s), else zlib."""
    if len(body) >= _DEVICE_CRC_MIN and _lib.cuda_available():
        torch = _lib.torch_cuda()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")  # read-only source buffer: only copied from
            t = torch.frombuffer(body, dtype=torch.uint8).cuda()
        return crc32_device(t, len(body))
    return zlib.crc32(body)


_side_streams: dict = {}


def _stream_pool(device, k):
    """Side streams; slot r has a higher priority than slot r+1 (torch maps
    the request onto the device's priority range)."""
    torch = _lib.torch_cuda()
    pool = _side_streams.setdefault(device, [])
    while len(pool) < k:
        pool.append(torch.cuda.Stream(device=device, priority=-(8 - len(pool))))
    return pool[:k]


def compress_batch(xs, params, max_concurrency: int = 8, ready=None, compact: bool = False, bit_hints=None):
    """Compress several fp32 CUDA tensors with ONE host synchronisation.

    Every tensor runs K1 (quantize/Lorenzo/histogram), K2 (codebook) and K3
    (encode) back to back on its own stream and context with no host round
    trip (actc_compress_async: the encoder reads its live symbol range from
    the device plan and writes into buffers sized by caps), so the
    single-CTA codebooks of some tensors overlap the bandwidth-bound kernels
    of others.  The plans are read after one synchronisation; a tensor that
    overflows a cap (or needs the > 26-bit encoder) is redone through the
    two-phase path.  Results are ordered on the caller's current stream.
    `ready` (optional, one CUDA event per tensor) lets each tensor start as
    soon as its own producer (e.g. its host-to-device copy) is done.
    `compact` copies the payload and outliers into exact-size buffers and
    releases the capped ones (stored activations, where memory is the point).
    `bit_hints` (optional, per tensor: expected payload bits or None) caps
    the payload at 1.25x the hint instead of n*ceil(log2 L) bits -- e.g. the
    same layer's previous size in training; an overflow is redone exactly.
    """
    torch = _lib.torch_cuda()
    if isinstance(params, CodecParams):
        params = [params] * len(xs)
    results = [None] * len(xs)
    # largest tensors first: the longest K1 -> K2 -> K3 chain starts earliest
    order = sorted(range(len(xs)), key=lambda i: -xs[i].numel())
    del torch
    for g0 in range(0, len(xs), max_concurrency):
        group = order[g0:g0 + max_concurrency]
        # a lone tensor runs on the caller's stream: no side-stream event
        # hand-offs on the host path (the call synchronises on it anyway)
        pend = compress_begin([xs[i] for i in group], [params[i] for i in group],
                              ready=None if ready is None else [ready[i] for i in group],
                              bit_hints=None if bit_hints is None else [bit_hints[i] for i in group],
                              on_caller_stream=len(xs) == 1 and ready is None)
        for i, r in zip(group, compress_end(pend, compact=compact)):
            results[i] = r
    return results


# tensors (element count, radius) whose frequency-class codebook needed the
# symbol-level fallback in an earlier async compression (diagnostics: every
# compression queues the fallback behind the frequency-class codebook -- a
# launch that exits at once unless it is needed -- because a tensor whose
# class count crosses the capacity mid-training would otherwise be redone
# synchronously, a multi-millisecond stall on the training stream)
_FALLBACK_SEEN: set = set()
# the last redos of compress_end (n, status, max_len, n_outliers, k_cap,
# payload_bits, cap_bits): why a launch overflowed a cap
REDOS: collections.deque = collections.deque(maxlen=64)


class PendingCompress:
    """Launched, not yet synchronised compressions (compress_begin)."""

    __slots__ = ("jobs", "main", "done", "events")

    def __init__(self, jobs, main):
        self.jobs = jobs
        self.main = main
        self.done = False
        self.events = [job[2].record_event() for job in jobs]  # each chain's end

    def ready(self) -> bool:
        """every compression of the batch has finished on the device (no wait)"""
        return all(e.query() for e in self.events)


def compress_begin(xs, params, slot_base: int = 0, ready=None, bit_hints=None,
                   own_scratch: bool = False, on_caller_stream: bool = False,
                   outlier_hints=None, queue_fallback: bool = True) -> PendingCompress:
    """Launch the compression of xs (each on its own side stream and context,
    slots slot_base .. slot_base+len-1) and return without synchronising;
    compress_end reads the plans and builds the containers.  The inputs are
    kept alive (and recorded on the side streams) until then, and the slots'
    contexts are busy: nothing else may use them (slot 0 is the thread's main
    context, used by compress_device / decompress_device) before compress_end.
    `own_scratch`: the symbol scratch (2-4 bytes per element) comes from
    torch's allocator per call and is released at compress_end, instead of
    the context's persistent buffer (memory-bound callers such as the hooks).
    `on_caller_stream`: the launches go on the caller's current stream (in
    order with its other work) instead of side streams.
    `outlier_hints` (optional, per tensor: expected outlier count or None)
    raises the outlier cap (default max(4096, n/64)) to 4x the hint + n/64
    -- small error bounds can put several percent of the elements outside
    the quantization radius, and a training activation's tail can grow
    several-fold in one step; an overflow is redone exactly.
    `queue_fallback=False` skips the (gated) symbol-level codebook launch
    (ACTC_ASYNC_NO_FALLBACK): a tensor that needs it is then redone."""
    torch = _lib.torch_cuda()
    if isinstance(params, CodecParams):
        params = [params] * len(xs)
    xs = [x if x.is_contiguous() else x.contiguous() for x in xs]
    for x in xs:
        if x.dtype != torch.float32:
            raise ParameterError("compress expects a 32-bit tensor; convert explicitly with astype(4)")
    dev_index = xs[0].device.index if xs else torch.cuda.current_device()
    main = _lib.current_stream()
    L = _lib.lib()
    streams = [main] * len(xs) if on_caller_stream else _stream_pool(dev_index, slot_base + len(xs))[slot_base:]
    jobs = []
    for j, (x, p) in enumerate(zip(xs, params)):
        s = streams[j]
        ctx = _lib.context_for(dev_index, slot_base + j)
        n = x.numel()
        if n == 0:
            raise ParameterError("empty tensor")
        nchunks = (n + _lib.ACTC_CHUNK - 1) // _lib.ACTC_CHUNK
        lmax = min(p.alphabet_size, n)
        cap_bits = n * max(1, (lmax - 1).bit_length())  # Huffman <= fixed-length code
        if bit_hints is not None and bit_hints[j]:
            cap_bits = min(cap_bits, int(bit_hints[j] * 1.25) + 4096)
        cap = _payload_buffer_bytes(cap_bits)
        k_cap = max(4096, n // 64)
        if outlier_hints is not None and outlier_hints[j]:
            k_cap = min(n, max(k_cap, 4 * int(outlier_hints[j]) + n // 64))
        dev = _DevBufs()
        # fixed-size arrays, and the capped (data-dependent) ones apart so
        # `compact` can replace the latter by exact-size copies
        fixed = dev.carve(x.device, [("chunk_lat", nchunks, 8), ("chunk_off", nchunks, 8),
                                     ("len_counts", 64, 4), ("table", _lib.ACTC_TABLE_BYTES, 1)])
        fp, of = fixed.data_ptr(), dev.offsets
        # data-dependent sizes (capped; `compact` copies their live extent)
        capped = dev.carve(x.device, [("out_idx", k_cap, 8), ("payload", cap, 1), ("out_val", k_cap, 4),
                                      ("canon", lmax, 4)])
        cp, oc = capped.data_ptr(), dev.offsets
        symbuf = None
        if own_scratch:
            sb = 2 if 2 * int(p.radius) <= 65536 else 4
            symbuf = torch.empty(sb * n + 64, dtype=torch.uint8, device=x.device)
            _lib.raise_for(L.actc_ctx_set_scratch(ctx.handle, symbuf.data_ptr(), symbuf.numel()))
        # recorded after this tensor's allocations: its side stream is ordered
        # after all caller-stream work that used the blocks the allocator reused
        if s is not main:
            s.wait_event(main.record_event())
        if ready is not None:
            s.wait_event(ready[j])
        flags = _lib.ACTC_FLAG_PRESERVE_ZEROS if p.preserve_zeros else 0
        if not queue_fallback:
            flags |= _lib.ACTC_ASYNC_NO_FALLBACK
        args = (ctx.handle, x.data_ptr(), n, float(p.eb), int(p.radius), flags, fp + of["chunk_lat"],
                cp + oc["payload"], cap, cp + oc["out_idx"], cp + oc["out_val"], k_cap, cp + oc["canon"],
                fp + of["len_counts"], fp + of["chunk_off"], ctx.plan_buf.data_ptr(), s.cuda_stream)
        # the whole chain (K1 -> codebook -> count -> pack) goes out in one
        # call: launching every tensor's K1 first held the first tensor's
        # codebook -- the batch's critical path -- back by the other tensors'
        # host preparation (~55 us each)
        # the chain's tail builds the stream's decode table into the container
        _lib.raise_for(L.actc_ctx_set_table_out(ctx.handle, dev.ptr("table"), _lib.ACTC_TABLE_BYTES))
        _lib.raise_for(L.actc_compress_async(*args))
        if s is not main:
            fixed.record_stream(s)
            capped.record_stream(s)
            x.record_stream(s)
            if symbuf is not None:
                symbuf.record_stream(s)
        jobs.append((x, p, s, ctx, dev, cap, k_cap, args, symbuf))
    return PendingCompress(jobs, main)


def compress_end(pend: PendingCompress, compact: bool = False, order: bool = True):
    """Synchronise a compress_begin batch: [(CompressedActivation, report)]
    in input order.  A tensor whose plan overflowed a cap is redone through
    the two-phase path (its input is still held).  With order=True the
    caller's stream is ordered after the compressions; with order=False it
    is not (training keeps computing): each container carries an event its
    readers wait for instead (decompress_* on the device, host reads on the
    host)."""
    if pend.done:
        raise ParameterError("compress_end called twice on the same batch")
    pend.done = True
    out = []
    redone = set()
    # containers are built as each stream finishes (the host work of the
    # early tensors overlaps the GPU tail of the late ones), and each
    # container's stream descriptor is built once here
    for x, p, s, ctx, dev, cap, k_cap, _, _sym in pend.jobs:
        s.synchronize()
        plan = _lib.Plan.from_buffer_copy(ctx.plan)
        n = x.numel()
        dims = tuple(x.shape) or (1,)
        fits = (plan.status == 0 and plan.max_len <= 56 and plan.n_outliers <= k_cap
                and plan.payload_bits <= 8 * (cap - 32))
        if fits:
            k = plan.n_outliers
            dev.shrink("out_idx", k)
            dev.shrink("out_val", k)
            dev.shrink("payload", _payload_buffer_bytes(plan.payload_bits))
            dev.shrink("canon", max(plan.live_symbols, 1))
            if compact:
                dev.compact(("out_idx", "payload", "out_val", "canon"), s, pend.main)
            c, rep = _container(n, p, dims, plan, dev)
            c._desc()
        else:
            REDOS.append((n, int(plan.status), int(plan.max_len), int(plan.n_outliers), k_cap,
                          int(plan.payload_bits), 8 * (cap - 32)))
            if plan.status == _lib.ACTC_EAGAIN:
                _FALLBACK_SEEN.add((n, int(p.radius)))  # next time: queue the fallback codebook
            else:
                _check_plan(plan)
            # the two-phase redo runs on the thread's main context: order it
            # after the caller's queued work (which may use that context) and
            # allocate on the stream it runs on
            torch = _lib.torch_cuda()
            s.wait_stream(pend.main)
            redone.add(s)
            with torch.cuda.stream(s):
                c, rep = compress_device(x, p)
        if not order:
            c._ready = s.record_event()
        out.append((c, rep))
    if order:
        # every chain has completed (its stream was synchronised above), so
        # only work queued after that -- compaction copies, redos -- needs
        # the caller's stream to wait
        for job in pend.jobs:
            if compact or job[2] in redone:
                pend.main.wait_stream(job[2])
    pend.jobs = []
    return out


def compress(t, params: CodecParams):
    """Compress a 32-bit tensor; returns (CompressedActivation, report).  codec.py:296-340."""
    torch = _lib.torch_cuda()
    if isinstance(t, torch.Tensor):
        return compress_device(to_device(t), params)
    if t.precision != 4:
        raise ParameterError("compress expects a 32-bit tensor; convert explicitly with astype(4)")
    return compress_device(to_device(t), params, dims=t.dims)


def decompress_device(c: CompressedActivation, dtype=None, out=None, stream=None, check=True,
                      count_nonzero=True, slot: int = 0):
    """Reconstruct on the device.  Returns (tensor, nonzero_count or None).

    dtype torch.float64 is bit-identical to the reference's output; float32
    stores fp32 of it.  With check=False no host synchronisation happens
    (the status and nonzero count are left in the context's mailbox).  With
    count_nonzero=False the decoder skips the nonzero count (R,
    training.py:351-352) and None is returned in its place.  `slot` picks
    the library context (0: the thread's main one; another slot for a
    decode running concurrently on another stream).
    """
    torch = _lib.torch_cuda()
    dtype = torch.float32 if dtype is None else dtype
    n = c.element_count
    if c.symbol_count != n:
        raise FormatError(f"symbol count {c.symbol_count} != element count {n}")
    c._ensure_index()
    dev = c.device
    ctx = _lib.context_for(dev.index, slot)
    sh, s = _lib.stream_handle(stream, dev)
    if out is None:
        with torch.cuda.stream(s):  # stream-ordered for the decoding stream
            out = torch.empty(c.dims, dtype=dtype, device=dev)
    code = _lib.ACTC_DTYPE_F32 if out.dtype == torch.float32 else _lib.ACTC_DTYPE_F64
    if out.dtype not in (torch.float32, torch.float64) or out.numel() != n or not out.is_contiguous():
        raise ParameterError("output must be a contiguous fp32/fp64 tensor with the stream's element count")
    d = c._desc()
    c._wait_ready(s)
    if not count_nonzero:
        code |= _lib.ACTC_DEC_NO_NONZERO
    _lib.raise_for(_lib.lib().actc_decompress(ctx.handle, C.byref(d), C.c_void_p(out.data_ptr()), code,
                                               C.c_void_p(ctx.dres_buf.data_ptr()), sh))
    if stream is not None:
        c._record_stream(s)  # the container is read on `s` (caching allocator)
    if not check:
        return out, None
    s.synchronize()
    r = _lib.DecodeResult.from_buffer_copy(ctx.dres)
    if r.status or r.markers != c._n_outliers:
        # reported here: the context's sticky fault word is collected too
        _lib.decode_status_result(_lib.take_decode_status(dev.index, s))
        if r.status:
            raise FormatError("invalid code in bitstream or outlier markers disagree with stored indices")
        raise FormatError("outlier markers disagree with stored indices")
    return out, (int(r.nonzero) if count_nonzero else None)


def _decode_rest(L, i, c, out, d, s, ctx, dt, evs):
    """queue stream i's decoder on side stream s (no result mailbox: nothing is read back)"""
    rc = L.actc_decompress(ctx.handle, C.byref(d), out.data_ptr(), dt | _lib.ACTC_DEC_REST, None, s.cuda_stream)
    if rc:
        _lib.raise_for(rc)
    out.record_stream(s)
    c._record_stream(s)
    if evs is not None:
        evs[i] = s.record_event()


def decompress_batch(cs, outs=None, dtype=None, max_concurrency: int = 8, done=None):
    """Reconstruct several streams concurrently, each on its own stream and
    context (a small tensor's decode alone does not fill the GPU).  Results
    are ordered on the caller's current stream; no host synchronisation: decode
    faults are collected by `check_decode_status` (one sync for many batches).
    If `done` is a list, it receives one CUDA event per stream (input order)
    recorded when that reconstruction is complete.
    """
    torch = _lib.torch_cuda()
    dtype = torch.float32 if dtype is None else dtype
    if outs is None:
        outs = [torch.empty(c.dims, dtype=dtype, device="cuda") for c in cs]
    if not cs:
        return outs
    dev_index = outs[0].device.index
    main = _lib.current_stream()
    order = sorted(range(len(cs)), key=lambda i: -cs[i].element_count)  # largest first
    evs = [None] * len(cs)
    for g0 in range(0, len(cs), max_concurrency):
        group = order[g0:g0 + max_concurrency]
        # a lone stream decodes on the caller's stream (no event hand-offs)
        streams = [main] if len(cs) == 1 else _stream_pool(dev_index, len(group))
        L = _lib.lib()
        f32 = torch.float32
        # uploads / index rebuilds of containers parsed from bytes run first,
        # on the caller's stream and the thread's main context -- which slot
        # 0's decoder uses too, so none may run while a decoder of the group
        # is already queued
        descs = {}
        for i in group:
            c, out = cs[i], outs[i]
            n = c.symbol_count
            if out.numel() != n or out.dtype not in (f32, torch.float64) or not out.is_contiguous():
                raise ParameterError("output must be a contiguous fp32/fp64 tensor with the stream's element count")
            d = c._desc_cache
            if d is None:
                if n != c.element_count:
                    raise FormatError(f"symbol count {n} != element count {c.element_count}")
                c._ensure_index()
                d = c._desc()
            descs[i] = d
        ready = main.record_event() if streams[0] is not main else None  # side streams follow the caller
        jobs = []
        for slot, i in enumerate(group):
            c, out, d = cs[i], outs[i], descs[i]
            s = streams[slot]
            if ready is not None:
                s.wait_event(ready)
            c._wait_ready(s)
            ctx = _lib.context_for(dev_index, slot)
            dt = _lib.ACTC_DTYPE_F32 if out.dtype == f32 else _lib.ACTC_DTYPE_F64
            if not d.table_dev:
                # every decode table goes out before any table-less stream's
                # decoder fills the GPU
                rc = L.actc_decompress(ctx.handle, C.byref(d), out.data_ptr(), dt | _lib.ACTC_DEC_LUT_ONLY,
                                       None, s.cuda_stream)
                if rc:
                    _lib.raise_for(rc)
                jobs.append((i, c, out, d, s, ctx, dt))
            else:
                # streams from compress_batch carry their decode table: the
                # decoder goes out at once (the GPU would idle until the first
                # one is queued; the host prepares the next while it runs)
                _decode_rest(L, i, c, out, d, s, ctx, dt, evs if done is not None else None)
        for i, c, out, d, s, ctx, dt in jobs:
            _decode_rest(L, i, c, out, d, s, ctx, dt, evs if done is not None else None)
        for slot in range(len(group)):
            if streams[slot] is not main:
                main.wait_stream(streams[slot])
    if done is not None:
        done.extend(evs)
    return outs


def check_decode_status(device=None):
    """Raise FormatError if any decompression issued by this thread on
    `device` since the last check met an invalid stream (bad code, stream
    length mismatch, outlier markers that disagree with the stored indices;
    huffman.py:228-235, codec.py:356-359).  `decompress_batch` does not
    synchronise; this is its check, one host synchronisation for all."""
    if _lib.decode_status_result(_lib.take_decode_status(device)):
        raise FormatError("invalid code in bitstream or outlier markers disagree with stored indices")


def decompress(c: CompressedActivation) -> Tensor:
    """Reconstruct the tensor a container describes (codec.py:343-369): fp64 host Tensor."""
    torch = _lib.torch_cuda()
    out, _ = decompress_device(c, dtype=torch.float64)
    return Tensor(out.cpu().numpy().reshape(c.dims), precision=8)


def write_compressed(c: CompressedActivation, sink) -> int:
    blob = c.to_bytes()
    if isinstance(sink, (str, bytes)) or hasattr(sink, "__fspath__"):
        with open(sink, "wb") as fh:
            fh.write(blob)
    else:
        sink.write(blob)
    return len(blob)


def read_compressed(source) -> CompressedActivation:
    if isinstance(source, (str, bytes)) or hasattr(source, "__fspath__"):
        with open(source, "rb") as fh:
            return CompressedActivation.from_bytes(fh.read())
    return CompressedActivation.from_bytes(source.read())


# ---------------------------------------------------------------------------
# pipeline internals (conformance entry points, all on the GPU)
# ---------------------------------------------------------------------------


def prequantize(t, eb: float) -> np.ndarray:
    """codec.py:238-251 on the GPU (exact fp64 path)."""
    if not (eb > 0 and np.isfinite(eb)):
        raise ParameterError(f"eb must be a positive finite real, got {eb}")
    torch = _lib.torch_cuda()
    data = t.data if isinstance(t, Tensor) else np.asarray(t)
    x = to_device(np.ascontiguousarray(data.reshape(-1)))
    if x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float64)
    q = torch.empty(x.numel(), dtype=torch.int64, device="cuda")
    sh, s = _lib.stream_handle()
    code = _lib.ACTC_DTYPE_F32 if x.dtype == torch.float32 else _lib.ACTC_DTYPE_F64
    _lib.raise_for(_lib.lib().actc_prequantize(C.c_void_p(x.data_ptr()), code, x.numel(), float(eb),
                                                C.c_void_p(q.data_ptr()), sh))
    return q.cpu().numpy()


def lorenzo_encode(lattice, radius: int, force_outlier=None):
    """codec.py:254-272 on the GPU: returns (symbols, outlier_indices)."""
    if radius < 2:
        raise ParameterError(f"radius must be >= 2, got {radius}")
    torch = _lib.torch_cuda()
    lat = to_device(np.ascontiguousarray(np.asarray(lattice, dtype=np.int64).reshape(-1)))
    n = lat.numel()
    sym = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    force = None
    if force_outlier is not None:
        force = to_device(np.ascontiguousarray(np.asarray(force_outlier, dtype=np.uint8).reshape(-1)))
    ctx = _lib.context()
    sh, s = _lib.stream_handle()
    _lib.raise_for(_lib.lib().actc_lorenzo_encode(
        C.c_void_p(lat.data_ptr()), n, int(radius), C.c_void_p(force.data_ptr()) if force is not None else None,
        C.c_void_p(sym.data_ptr()), C.c_void_p(ctx.u64_buf.data_ptr()), sh))
    s.synchronize()
    symbols = sym[:n].cpu().numpy().view(np.uint32).astype(np.int64)
    return symbols, np.flatnonzero(symbols == 0).astype(np.int64)


def lorenzo_decode(symbols, outlier_lattice, radius: int) -> np.ndarray:
    """codec.py:275-293 on the GPU."""
    torch = _lib.torch_cuda()
    s_h = np.asarray(symbols, dtype=np.int64).reshape(-1)
    n = s_h.size
    sym = to_device(np.ascontiguousarray(s_h.astype(np.uint32).view(np.int32)))
    ol = np.asarray(outlier_lattice, dtype=np.int64).reshape(-1)
    olat = to_device(np.ascontiguousarray(ol)) if ol.size else torch.zeros(1, dtype=torch.int64, device="cuda")
    out = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    ctx = _lib.context()
    sh, s = _lib.stream_handle()
    _lib.raise_for(_lib.lib().actc_lorenzo_decode(
        C.c_void_p(sym.data_ptr()), n, C.c_void_p(olat.data_ptr()), ol.size, int(radius),
        C.c_void_p(out.data_ptr()), C.c_void_p(ctx.u64_buf.data_ptr()), sh))
    s.synchronize()
    if int(ctx.u64_buf[:4].view(torch.int32).item()):
        n_markers = int(np.count_nonzero(s_h == 0))
        raise FormatError(f"outlier count mismatch: {n_markers} markers, {ol.size} stored values")
    return out[:n].cpu().numpy()
