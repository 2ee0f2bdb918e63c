"""GPU parity: the CUDA path against the reference-generated golden vectors
and the C oracle (bit-exact codes, bitstreams, CMTZ bytes, ratio, fp64
reconstruction; fp32 output == fp32(reference fp64))."""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import codec as pc  # noqa: E402
from paper_2111_09562_b200.errors import DataError, FormatError, ParameterError  # noqa: E402


def _params(m):
    return pb.CodecParams(eb=m["eb"], radius=m["radius"], preserve_zeros=m["preserve"])


def test_golden_blobs_and_reports(codec_golden, golden_meta):
    for m in golden_meta["codec"]:
        i = m["i"]
        x = codec_golden[f"x_{i}"]
        c, rep = pb.compress(pb.Tensor(x), _params(m))
        assert c.to_bytes() == codec_golden[f"blob_{i}"].tobytes(), m["name"]
        assert rep.compressed_bytes == m["compressed_bytes"], m["name"]
        assert rep.ratio == m["ratio"], m["name"]
        assert rep.outlier_fraction == m["outlier_fraction"], m["name"]
        assert rep.outlier_warning == m["outlier_warning"], m["name"]
        assert abs(rep.codes_entropy_bits_per_symbol - m["entropy"]) <= 1e-12 * max(1.0, m["entropy"]), m["name"]
        assert c.payload_bits == m["payload_bits"], m["name"]


def test_golden_reconstruction_fp64_and_fp32(codec_golden, golden_meta):
    for m in golden_meta["codec"]:
        i = m["i"]
        x = codec_golden[f"x_{i}"]
        c, _ = pb.compress(pb.Tensor(x), _params(m))
        back = pb.decompress(c)
        assert back.precision == 8 and back.dims == x.shape
        assert hashlib.sha256(np.ascontiguousarray(back.data).tobytes()).hexdigest() == m["recon_sha256"], m["name"]
        if m["recon_stored"]:
            ref = codec_golden[f"recon_{i}"]
            out32, nz = pb.decompress_device(c, dtype=torch.float32)
            got = out32.cpu().numpy().reshape(-1)
            # contract: fp32 output is fp32(reference fp64), i.e. 0 ulp
            assert np.array_equal(got.view(np.uint32), ref.astype(np.float32).view(np.uint32)), m["name"]
            assert nz == int(np.count_nonzero(ref)), m["name"]


def test_golden_blob_decode_via_from_bytes(codec_golden, golden_meta):
    """blobs from disk carry no chunk index: exercised the self-sync rebuild."""
    for m in golden_meta["codec"]:
        i = m["i"]
        blob = codec_golden[f"blob_{i}"].tobytes()
        c = pc.CompressedActivation.from_bytes(blob)
        back = pb.decompress(c)
        assert hashlib.sha256(np.ascontiguousarray(back.data).tobytes()).hexdigest() == m["recon_sha256"], m["name"]
        assert c.to_bytes() == blob


@pytest.mark.parametrize("rel", [1e-1, 1e-2, 1e-3, 1e-4])
def test_config1_full_size_vs_oracle(oracle, rel):
    x = np.maximum(np.random.default_rng(0).normal(0, 1, 32 * 64 * 56 * 56), 0).astype(np.float32).reshape(32, 64, 56, 56)
    eb = rel * float(x.max() - x.min())
    ref = oracle.compress(x, eb, debug=False)
    c, rep = pb.compress(pb.Tensor(x), pb.CodecParams(eb=eb))
    assert c.to_bytes() == ref.blob
    assert rep.ratio == ref.ratio
    want = oracle.decompress_blob(ref.blob, x.size)
    out, nz = pb.decompress_device(c, dtype=torch.float64)
    assert np.array_equal(out.cpu().numpy().reshape(-1).view(np.uint64), want.view(np.uint64))
    assert nz == int(np.count_nonzero(want))
    if rel == 1e-2:
        assert round(rep.ratio, 3) == 6.982  # SURVEY 8d measured oracle ratio


def test_device_input_and_errors():
    x = torch.randn(1000, device="cuda").relu()
    c, rep = pb.compress(x, pb.CodecParams(eb=1e-3))
    out, _ = pb.decompress_device(c)
    # fp32(reference fp64 recon): |x - x_hat| <= eb + ulp(x_hat)/2, or a re-zeroed |x| <= 2 eb
    half_ulp = (torch.nextafter(out.abs(), torch.full_like(out, float("inf"))) - out.abs()).double() / 2
    err = (x.double() - out.double()).abs()
    assert bool(((err <= 1e-3 + half_ulp) | ((out == 0) & (x.abs().double() <= 2e-3))).all())
    with pytest.raises(ParameterError):
        pb.compress(x.double(), pb.CodecParams(eb=1e-3))
    bad = x.clone()
    bad[17] = float("nan")
    with pytest.raises(DataError):
        pb.compress(bad, pb.CodecParams(eb=1e-3))
    with pytest.raises(ParameterError):
        pb.compress(pb.make_tensor([8], "uniform", seed=0, precision=8), pb.CodecParams(eb=1e-3))


def test_bound_and_zero_fidelity_random_sizes():
    rng = np.random.default_rng(20240501)
    for trial in range(60):
        n = int(10 ** rng.uniform(0, 6))
        eb = (1e-2, 1e-3, 1e-4)[trial % 3]
        kind = trial % 3
        if kind == 0:
            data = rng.uniform(-1, 1, n)
        elif kind == 1:
            data = rng.normal(0, 1, n)
        else:
            data = np.maximum(rng.normal(0, 1, n), 0.0)
        t = pb.Tensor(data.astype(np.float32))
        back = pb.decompress(pb.compress(t, pb.CodecParams(eb=eb))[0])
        xx = t.data.astype(np.float64)
        xh = back.data
        ok = (np.abs(xx - xh) <= eb) | ((xh == 0.0) & (np.abs(xx) <= 2.0 * eb))
        assert ok.all(), (n, eb)
        assert np.all(xh[xx == 0.0] == 0.0)


def test_random_sizes_bit_exact_vs_oracle(oracle):
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(10 ** rng.uniform(0, 5.5))
        data = (np.maximum(rng.normal(0, 1, n), 0) if trial % 2 else rng.normal(0, 3, n)).astype(np.float32)
        eb = float(10 ** rng.uniform(-5, -1))
        radius = int(rng.choice([2, 7, 512, 1 << 15, 1 << 17]))
        ref = oracle.compress(data, eb, radius, trial % 5 != 0)
        c, rep = pb.compress(pb.Tensor(data), pb.CodecParams(eb=eb, radius=radius, preserve_zeros=trial % 5 != 0))
        assert c.to_bytes() == ref.blob, (trial, n, eb, radius)
        want = oracle.decompress_blob(ref.blob, n)
        assert np.array_equal(pb.decompress(c).data.view(np.uint64), want.view(np.uint64)), (trial, n, eb, radius)


def test_container_crc_and_truncation(codec_golden, golden_meta):
    m = golden_meta["codec"][1]
    blob = bytearray(codec_golden[f"blob_{m['i']}"].tobytes())
    rng = np.random.default_rng(7)
    for _ in range(50):
        pos = int(rng.integers(0, len(blob) * 8))
        blob[pos // 8] ^= 1 << (pos % 8)
        with pytest.raises(FormatError):
            pc.CompressedActivation.from_bytes(bytes(blob))
        blob[pos // 8] ^= 1 << (pos % 8)
    with pytest.raises(FormatError):
        pc.CompressedActivation.from_bytes(bytes(blob[: len(blob) // 2]))


def test_corrupt_payload_is_format_error():
    x = np.maximum(np.random.default_rng(3).normal(0, 1, 20000), 0).astype(np.float32)
    c, _ = pb.compress(pb.Tensor(x), pb.CodecParams(eb=1e-3))
    blob = bytearray(c.to_bytes())
    # flip payload bits and fix the CRC so only the bitstream is wrong
    import struct
    import zlib

    hits = 0
    for pos in (200, 500, 800):
        b = bytearray(blob)
        b[pos] ^= 0xFF
        b[-4:] = struct.pack("<I", zlib.crc32(bytes(b[:-4])))
        try:
            back = pb.decompress(pc.CompressedActivation.from_bytes(bytes(b)))
        except FormatError:
            hits += 1
    assert hits >= 1


@pytest.mark.parametrize("eb", [1.2e-6, 6.3e-6, 3.7e-5])
def test_small_eb_outlier_heavy_vs_oracle(oracle, eb):
    """the adaptive bounds of AlexNet's deeper layers at init: deltas exceed
    the radius, so a large share of elements are outliers"""
    rng = np.random.default_rng(int(eb * 1e9))
    x = (np.maximum(rng.normal(0, 0.05, (16, 256, 13, 13)), 0)).astype(np.float32)
    ref = oracle.compress(x, eb, debug=False)
    c, rep = pb.compress(pb.Tensor(x), pb.CodecParams(eb=eb))
    assert c.to_bytes() == ref.blob
    assert rep.ratio == ref.ratio
    want = oracle.decompress_blob(ref.blob, x.size)
    out, nz = pb.decompress_device(c, dtype=torch.float64)
    assert np.array_equal(out.cpu().numpy().reshape(-1).view(np.uint64), want.view(np.uint64))
    out32, _ = pb.decompress_device(c, dtype=torch.float32)
    assert np.array_equal(out32.cpu().numpy().reshape(-1), want.astype(np.float32))


def test_compress_batch_matches_single(oracle):
    rng = np.random.default_rng(17)
    xs, ps = [], []
    for k in range(11):
        n = int(rng.integers(1, 300000))
        xs.append(torch.from_numpy(np.maximum(rng.normal(0, 1, n), 0).astype(np.float32)).cuda())
        ps.append(pb.CodecParams(eb=float(10 ** rng.uniform(-5, -1))))
    out = pb.compress_batch(xs, ps, max_concurrency=4)
    for (c, rep), x, p in zip(out, xs, ps):
        ref = oracle.compress(x.cpu().numpy(), p.eb, debug=False)
        assert c.to_bytes() == ref.blob
        assert rep.ratio == ref.ratio
        back, _ = pb.decompress_device(c, dtype=torch.float64)
        want = oracle.decompress_blob(ref.blob, x.numel())
        assert np.array_equal(back.cpu().numpy().view(np.uint64), want.view(np.uint64))


def test_decompress_batch_matches_single(oracle):
    rng = np.random.default_rng(23)
    xs, ps = [], []
    for k in range(6):
        n = int(rng.integers(1, 400000))
        xs.append(torch.from_numpy(np.maximum(rng.normal(0, 1, n), 0).astype(np.float32)).cuda())
        ps.append(pb.CodecParams(eb=float(10 ** rng.uniform(-6, -1))))
    comp = pb.compress_batch(xs, ps, max_concurrency=3)
    outs = pb.decompress_batch([c for c, _ in comp], max_concurrency=3)
    outs64 = pb.decompress_batch([c for c, _ in comp], dtype=torch.float64)
    torch.cuda.synchronize()
    for (c, rep), x, p, o, o64 in zip(comp, xs, ps, outs, outs64):
        want = oracle.decompress_blob(oracle.compress(x.cpu().numpy(), p.eb, debug=False).blob, x.numel())
        assert np.array_equal(o64.cpu().numpy().reshape(-1).view(np.uint64), want.view(np.uint64))
        assert np.array_equal(o.cpu().numpy().reshape(-1), want.astype(np.float32))


def test_decompress_batch_mixed_table_and_blob_streams(oracle):
    """a batch mixing containers that carry the pack kernel's decode table
    (decoded as soon as prepared) with containers parsed from bytes (table
    first, decoder after every table): every reconstruction bit-exact, and
    one completion event per stream in input order"""
    rng = np.random.default_rng(31)
    xs, ps = [], []
    for k in range(7):
        n = int(rng.integers(1000, 300000))
        xs.append(torch.from_numpy(np.maximum(rng.normal(0, 1, n), 0).astype(np.float32)).cuda())
        ps.append(pb.CodecParams(eb=float(10 ** rng.uniform(-5, -2))))
    comp = [c for c, _ in pb.compress_batch(xs, ps)]
    mixed = [c if k % 2 == 0 else pc.CompressedActivation.from_bytes(c.to_bytes()) for k, c in enumerate(comp)]
    done = []
    outs = pb.decompress_batch(mixed, max_concurrency=4, done=done)
    assert len(done) == len(mixed) and all(e is not None for e in done)
    for e in done:
        e.synchronize()
    pb.check_decode_status()
    for x, p, o in zip(xs, ps, outs):
        want = oracle.decompress_blob(oracle.compress(x.cpu().numpy(), p.eb, debug=False).blob, x.numel())
        assert np.array_equal(o.cpu().numpy().reshape(-1), want.astype(np.float32))


def test_compress_async_split_launch_matches_oracle(oracle):
    """the C ABI's split form of actc_compress_async (ACTC_ASYNC_K1_ONLY, then
    ACTC_ASYNC_REST on the same context and stream) gives the one-call
    result: every blob equal to the oracle's"""
    from paper_2111_09562_b200 import _lib

    L = _lib.lib()
    one_call = L.actc_compress_async

    def split(*args):
        rc = one_call(*args[:5], args[5] | _lib.ACTC_ASYNC_K1_ONLY, *args[6:])
        if rc:
            return rc
        return one_call(*args[:5], args[5] | _lib.ACTC_ASYNC_REST, *args[6:])

    rng = np.random.default_rng(37)
    xs = [torch.from_numpy(np.maximum(rng.normal(0, 1, int(n)), 0).astype(np.float32)).cuda()
          for n in rng.integers(1000, 200000, 4)]
    ps = [pb.CodecParams(eb=float(10 ** rng.uniform(-5, -2))) for _ in xs]
    L.actc_compress_async = split
    try:
        out = pb.compress_batch(xs, ps)
    finally:
        L.actc_compress_async = one_call
    for (c, rep), x, p in zip(out, xs, ps):
        assert c.to_bytes() == oracle.compress(x.cpu().numpy(), p.eb, debug=False).blob


def test_compress_batch_cap_overflow_takes_two_phase_path(oracle):
    """actc_compress_async sizes outlier buffers by a cap (max(4096, n/64));
    a tensor with more outliers must come back through the two-phase path,
    bit-exact either way"""
    rng = np.random.default_rng(29)
    n = 200_000
    x = (rng.standard_normal(n) * 1e4).astype(np.float32)  # deltas >> radius at this eb: ~all outliers
    small = np.maximum(rng.normal(0, 1, 50_000), 0).astype(np.float32)
    xs = [torch.from_numpy(x).cuda(), torch.from_numpy(small).cuda()]
    ps = [pb.CodecParams(eb=1e-3, radius=64), pb.CodecParams(eb=1e-2)]
    out = pb.compress_batch(xs, ps)
    for (c, rep), xt, p in zip(out, xs, ps):
        ref = oracle.compress(xt.cpu().numpy(), p.eb, radius=p.radius, debug=False)
        assert c.to_bytes() == ref.blob
        assert rep.ratio == ref.ratio
    assert out[0][1].outlier_fraction > 0.5
    back = pb.decompress_batch([c for c, _ in out], dtype=torch.float64)
    torch.cuda.synchronize()
    for o, xt, p in zip(back, xs, ps):
        want = oracle.decompress_blob(oracle.compress(xt.cpu().numpy(), p.eb, radius=p.radius, debug=False).blob,
                                      xt.numel())
        assert np.array_equal(o.cpu().numpy().reshape(-1).view(np.uint64), want.view(np.uint64))


def test_compress_batch_compact(oracle):
    """compact=True: payload/outliers moved to exact-size buffers; same bytes"""
    rng = np.random.default_rng(31)
    xs = [torch.from_numpy(np.maximum(rng.normal(0, 1, n), 0).astype(np.float32)).cuda() for n in (70000, 300000)]
    ps = [pb.CodecParams(eb=1e-3), pb.CodecParams(eb=1e-5)]  # the second overflows the outlier cap
    loose = pb.compress_batch(xs, ps)
    tight = pb.compress_batch(xs, ps, compact=True)
    for (c0, r0), (c1, r1), x, p in zip(loose, tight, xs, ps):
        assert c1.to_bytes() == c0.to_bytes() == oracle.compress(x.cpu().numpy(), p.eb, debug=False).blob
        assert c1.device_nbytes <= c0.device_nbytes
    assert tight[0][0].device_nbytes < loose[0][0].device_nbytes
    outs = pb.decompress_batch([c for c, _ in tight], dtype=torch.float64)
    torch.cuda.synchronize()
    for o, x, p in zip(outs, xs, ps):
        want = oracle.decompress_blob(oracle.compress(x.cpu().numpy(), p.eb, debug=False).blob, x.numel())
        assert np.array_equal(o.cpu().numpy().reshape(-1).view(np.uint64), want.view(np.uint64))


def _fibonacci_deltas(rng, depth):
    """integer-valued signal whose Lorenzo deltas 0, 1, -1, 2, -2, ... occur
    with Fibonacci counts: a Huffman tree ~depth levels deep, its longest
    codes (> 26 bits) confined to a few segments"""
    fib = [1, 1]
    while len(fib) < depth:
        fib.append(fib[-1] + fib[-2])
    vals = [((i + 1) // 2) * (1 if i % 2 else -1) for i in range(depth)]
    d = np.repeat(np.array(vals, dtype=np.int64), fib[::-1])
    rng.shuffle(d)
    return np.cumsum(d).astype(np.float32)  # eb = 0.5: x / (2 eb) is exact


@pytest.mark.parametrize("depth", [29, 33])
def test_long_codes_bit_exact(oracle, depth):
    """codes longer than 26 bits take the segment encoder's u64 path (single
    and batched compress) and the decoders' long-code entries"""
    x = _fibonacci_deltas(np.random.default_rng(depth), depth)
    p = pb.CodecParams(eb=0.5)
    ref = oracle.compress(x, p.eb, debug=False)
    c, rep = pb.compress(pb.Tensor(x), p)
    assert 26 < int(c.code_lengths.max()) <= 56
    assert c.to_bytes() == ref.blob
    assert rep.ratio == ref.ratio
    xt = torch.from_numpy(x).cuda()
    (cb, _), = pb.compress_batch([xt], [p])
    assert cb.to_bytes() == ref.blob
    want = oracle.decompress_blob(ref.blob, x.size)
    for cc in (c, cb, pc.CompressedActivation.from_bytes(ref.blob)):
        out, _ = pb.decompress_device(cc, dtype=torch.float64)
        assert np.array_equal(out.cpu().numpy().reshape(-1).view(np.uint64), want.view(np.uint64))


def test_async_codebook_fallback_redo_and_memory(oracle):
    """> 6144 distinct symbol frequencies exceed the frequency-class codebook:
    without the fallback launch (queue_fallback=False) the compression sees
    ACTC_EAGAIN and is redone through the two-phase path; by default the
    gated symbol-level codebook runs on the device right behind it, no redo.
    Both bit-exact."""
    K = 6500
    rng = np.random.default_rng(1)
    vals = np.array([((i + 1) // 2) * (1 if i % 2 else -1) for i in range(K)], dtype=np.int64)
    d = np.repeat(vals, np.arange(K, 0, -1))
    rng.shuffle(d)
    x = np.cumsum(d).astype(np.float32)  # eb = 0.5: exact lattice values
    p = pb.CodecParams(eb=0.5)
    ref = oracle.compress(x, p.eb, debug=False)
    xt = torch.from_numpy(x).cuda()
    key = (x.size, p.radius)
    pc._FALLBACK_SEEN.discard(key)
    (c1, r1), = pc.compress_end(pc.compress_begin([xt], [p], queue_fallback=False))
    assert key in pc._FALLBACK_SEEN  # redone
    n0 = len(pc.REDOS)
    (c2, r2), = pb.compress_batch([xt], [p])
    assert len(pc.REDOS) == n0  # the device ran the fallback codebook
    for c, r in ((c1, r1), (c2, r2)):
        assert c.to_bytes() == ref.blob
        assert r.ratio == ref.ratio
    out = pb.decompress_batch([c2], dtype=torch.float64)[0]
    want = oracle.decompress_blob(ref.blob, x.size)
    assert np.array_equal(out.cpu().numpy().reshape(-1).view(np.uint64), want.view(np.uint64))


def test_compress_begin_end_with_caller_scratch(oracle):
    """compress_begin/compress_end (the hooks' path): launched without a host
    sync, symbol scratch from torch's allocator, private side slots; same
    bytes as the reference, and the decode table carried by the container
    reconstructs like a table built at decode time (from_bytes)."""
    rng = np.random.default_rng(41)
    xs = [np.maximum(rng.normal(0, 1, n), 0).astype(np.float32) for n in (300_001, 70_000, 5)]
    ps = [pb.CodecParams(eb=e) for e in (1e-3, 1e-5, 1e-2)]
    pend = [pc.compress_begin([torch.from_numpy(x).cuda()], [p], slot_base=1 + k, own_scratch=True)
            for k, (x, p) in enumerate(zip(xs, ps))]
    outs = [pc.compress_end(q, compact=True)[0] for q in pend]
    for (c, rep), x, p in zip(outs, xs, ps):
        ref = oracle.compress(x, p.eb, debug=False)
        assert c.to_bytes() == ref.blob and rep.ratio == ref.ratio
        want = oracle.decompress_blob(ref.blob, x.size)
        got = pb.decompress_batch([c], dtype=torch.float64)[0]
        again = pb.decompress_batch([pc.CompressedActivation.from_bytes(ref.blob)], dtype=torch.float64)[0]
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy().reshape(-1).view(np.uint64), want.view(np.uint64))
        assert np.array_equal(again.cpu().numpy().reshape(-1).view(np.uint64), want.view(np.uint64))
    assert outs[0][0]._desc().table_dev  # decode table built with the stream (async path)
    with pytest.raises(ParameterError):
        pc.compress_end(pend[0])
