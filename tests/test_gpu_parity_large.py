"""GPU parity on what the bench measures and at the sizes it runs:

* the AlexNet conv/ReLU activations at the controller's adaptive error bound
  (the headline workload's regime: 12-64 K live symbols, long codes);
* a 1 GiB relu-normal tensor at rel 1e-2 / 1e-4 (config-5 sweep cell);
* a 2^30-element tensor whose payload exceeds 2^32 bits (u64 offsets);
* the fp32 fast quantizer over every fp32 bit pattern;
* error parity: random payload corruptions raise FormatError exactly when
  the reference decoder raises (huffman.py:228-235, codec.py:356-359).

All against the C oracle (bit-exact restatement of the reference, pinned on
reference-generated golden vectors in tests/test_oracle_golden.py).
"""
import ctypes as C
import hashlib
import os
import struct
import sys
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import _lib  # noqa: E402
from paper_2111_09562_b200 import codec as pc  # noqa: E402
from paper_2111_09562_b200.errors import FormatError  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sha(b):
    return hashlib.sha256(b).hexdigest()


@pytest.mark.parametrize("eb", [0.053217172622680664, 1e-2, 2.1e-4, 1.2e-6, 3e-8, 0.5, 1e3])
def test_quant_fast_path_exhaustive_fp32(eb):
    """K1's fp32 multiply fast path (actc_internal.cuh quant_fast32, a margin
    argument) against the exact fp64 restatement for all 2^32 patterns."""
    out = torch.zeros(2, dtype=torch.int64).pin_memory()
    sh, s = _lib.stream_handle()
    _lib.raise_for(_lib.lib().actc_debug_quant_check(float(eb), 0, 1 << 32, C.c_void_p(out.data_ptr()), sh))
    s.synchronize()
    bad, fast = int(out[0]), int(out[1])
    assert bad == 0, f"{bad} fp32 patterns quantize differently on the fast path at eb={eb}"
    assert fast > (1 << 31)  # the fast path takes most finite patterns


def test_alexnet_adaptive_eb_activations_vs_oracle(oracle):
    """The benchmarked regime: AlexNet's five conv/ReLU outputs (batch 32) at
    the error bounds the controller plans from live statistics."""
    sys.path.insert(0, ROOT)
    import bench

    layers, ebs, info, _ = bench.alexnet_activations(batch=32, seed=0, device="cuda")
    ps = [pb.CodecParams(eb=e) for e in ebs]
    comp = pb.compress_batch(layers, ps)
    outs = pb.decompress_batch([c for c, _ in comp])
    torch.cuda.synchronize()
    pb.check_decode_status()
    live = []
    for (c, rep), x, p, o in zip(comp, layers, ps, outs):
        xh = x.cpu().numpy()  # shaped: the CMTZ header records the dims
        ref = oracle.compress(xh, p.eb, debug=False)
        assert c.to_bytes() == ref.blob
        assert rep.ratio == ref.ratio
        want = oracle.decompress_blob(ref.blob, xh.size)
        assert np.array_equal(o.reshape(-1).cpu().numpy().view(np.uint32), want.astype(np.float32).view(np.uint32))
        live.append(c._live)
    assert min(live) > 1000


def _relu_normal(n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(n, device="cuda", generator=g).clamp_min_(0)


@pytest.mark.parametrize("rel", [1e-2, 1e-4])
def test_1gib_tensor_vs_oracle(oracle, rel):
    n = 1 << 28  # 1 GiB of fp32
    x = _relu_normal(n, 1234)
    eb = rel * float((x.max() - x.min()).item())
    c, rep = pb.compress(x, pb.CodecParams(eb=eb))
    (cb, rb), = pb.compress_batch([x], [pb.CodecParams(eb=eb)])
    xh = x.cpu().numpy()
    ref = oracle.compress(xh, eb, debug=False)
    blob = c.to_bytes()
    assert len(blob) == len(ref.blob) == rep.compressed_bytes and rep.ratio == ref.ratio
    assert _sha(blob) == _sha(ref.blob)
    assert cb.to_bytes() == ref.blob and rb.ratio == ref.ratio
    want = oracle.decompress_blob(ref.blob, n).astype(np.float32)
    out = pb.decompress_batch([cb])[0]
    torch.cuda.synchronize()
    pb.check_decode_status()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))


def test_2p30_elements_payload_over_2p32_bits(oracle):
    """4 GiB of fp32 at rel 1e-4: ~10 bits per symbol, so bit offsets pass
    2^32 (the encoder's prefix sums, the decode index and the decoders all
    use 64-bit positions)."""
    n = 1 << 30
    x = _relu_normal(n, 99)
    eb = 1e-4 * float((x.max() - x.min()).item())
    (c, rep), = pb.compress_batch([x], [pb.CodecParams(eb=eb)])
    assert c.payload_bits > (1 << 32)
    xh = x.cpu().numpy()
    ref = oracle.compress(xh, eb, debug=False)
    assert ref.payload_bits == c.payload_bits and rep.ratio == ref.ratio
    assert _sha(c.to_bytes()) == _sha(ref.blob)
    out = pb.decompress_batch([c])[0]
    torch.cuda.synchronize()
    pb.check_decode_status()
    got = out.cpu().numpy().view(np.uint32)
    del out, c, x
    want = oracle.decompress_blob(ref.blob, n)
    step = 1 << 26
    for i in range(0, n, step):
        assert np.array_equal(got[i:i + step], want[i:i + step].astype(np.float32).view(np.uint32)), i


def _oracle_raises(oracle, blob, n):
    try:
        return False, oracle.decompress_blob(blob, n)
    except oracle.OracleError:
        return True, None


def test_error_parity_random_payload_corruption(oracle):
    """Random byte corruptions of the payload (CRC recomputed, so only the
    bitstream is wrong): the drop-in raises FormatError exactly when the
    reference decoder does, and otherwise reconstructs the same values."""
    rng = np.random.default_rng(5)
    x = np.maximum(rng.normal(0, 1, 40_000), 0).astype(np.float32)
    x[rng.integers(0, x.size, 40)] = 1e6  # a few outliers: marker checks take part
    eb = 1e-3
    ref = oracle.compress(x, eb, debug=False)
    blob = ref.blob
    pay_bytes = (ref.payload_bits + 7) // 8
    p0 = len(blob) - 4 - pay_bytes
    raised = agree = 0
    for trial in range(300):
        b = bytearray(blob)
        for _ in range(int(rng.integers(1, 4))):
            pos = p0 + int(rng.integers(0, pay_bytes))
            b[pos] ^= int(rng.integers(1, 256))
        b[-4:] = struct.pack("<I", zlib.crc32(bytes(b[:-4])))
        b = bytes(b)
        want_raise, want = _oracle_raises(oracle, b, x.size)
        try:
            got = pb.decompress(pc.CompressedActivation.from_bytes(b)).data.reshape(-1)
            got_raise = False
        except FormatError:
            got_raise = True
        assert got_raise == want_raise, trial
        if not got_raise:
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), trial
        raised += got_raise
        agree += 1
    assert raised > 100 and agree == 300


def test_error_parity_outlier_table(oracle):
    """Stored outlier indices that disagree with the marker positions."""
    rng = np.random.default_rng(6)
    x = np.maximum(rng.normal(0, 1, 10_000), 0).astype(np.float32)
    x[[10, 500, 9000]] = 1e6
    ref = oracle.compress(x, 1e-3, debug=False)
    assert ref.k >= 3  # each spike: the jump up and the jump back down
    # outlier pairs start right after the header: 21 + 8*rank + 8 (count)
    off = 21 + 8 + 8
    for j, newidx in ((0, 12), (1, 9001), (ref.k - 1, 9999)):
        b = bytearray(ref.blob)
        b[off + 12 * j: off + 12 * j + 8] = struct.pack("<Q", newidx)
        b[-4:] = struct.pack("<I", zlib.crc32(bytes(b[:-4])))
        want_raise, _ = _oracle_raises(oracle, bytes(b), x.size)
        assert want_raise
        with pytest.raises(FormatError):
            pb.decompress(pc.CompressedActivation.from_bytes(bytes(b)))


def test_batched_decode_fault_is_collected():
    """decompress_batch does not synchronise; a corrupted device payload is
    reported by check_decode_status (the sticky per-context status)."""
    x = torch.from_numpy(np.maximum(np.random.default_rng(8).normal(0, 1, 100_000), 0).astype(np.float32)).cuda()
    (c, _), = pb.compress_batch([x], [pb.CodecParams(eb=1e-3)])
    try:
        pb.check_decode_status()  # faults of earlier tests on this thread's contexts
    except FormatError:
        pass
    pb.decompress_batch([c])
    pb.check_decode_status()  # clean stream: no error
    c._dev["payload"][1000:1064] ^= 0x5A  # corrupt the device-resident bitstream
    pb.decompress_batch([c])
    with pytest.raises(FormatError):
        pb.check_decode_status()
    pb.check_decode_status()  # the status was collected and reset
