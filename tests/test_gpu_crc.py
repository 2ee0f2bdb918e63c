"""K6 device CRC-32 against zlib.crc32 (the CMTZ checksum, codec.py:118 and
:126): every length class around the piece (256 B) and block (64 KiB)
boundaries, misaligned starts, running values; and the container paths that
use it (to_bytes of device-resident streams, from_bytes of large blobs)."""
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import codec as pc  # noqa: E402
from paper_2111_09562_b200.errors import FormatError  # noqa: E402

LENGTHS = [0, 1, 2, 3, 4, 5, 7, 8, 15, 16, 17, 255, 256, 257, 4095, 8192, 65535, 65536, 65537,
           131072 + 13, 1 << 20, (1 << 20) + 3, 16 * 65536 * 256 + 5]


@pytest.mark.parametrize("n", LENGTHS)
def test_crc32_matches_zlib(n):
    rng = np.random.default_rng(n)
    host = rng.integers(0, 256, n + 64, dtype=np.uint8)
    dev = torch.from_numpy(host).cuda()
    for off in (0, 1, 5, 16) if n < (1 << 22) else (0, 3):
        data = host[off:off + n].tobytes()
        for value in (0, 0xFFFFFFFF, 0x12345678):
            got = pc.crc32_device(dev[off:], n, value)
            assert got == zlib.crc32(data, value), (n, off, value)


def test_crc32_zeros_and_patterns():
    for n in (1, 64, 70000, 3 << 20):
        for fill in (0, 0xFF, 0xA5):
            t = torch.full((n,), fill, dtype=torch.uint8, device="cuda")
            assert pc.crc32_device(t, n) == zlib.crc32(bytes([fill]) * n)


def test_to_bytes_device_crc_equals_host_serialisation(oracle):
    rng = np.random.default_rng(7)
    x = np.maximum(rng.normal(0, 1, (64, 64, 56, 56)), 0).astype(np.float32)  # ~50 MB payload class
    eb = 1e-3 * float(x.max() - x.min())
    c, _ = pb.compress(pb.Tensor(x), pb.CodecParams(eb=eb))
    assert c.is_device_resident
    blob = c.to_bytes()
    assert blob == oracle.compress(x, eb, debug=False).blob
    assert zlib.crc32(blob[:-4]) == int.from_bytes(blob[-4:], "little")


def test_from_bytes_large_blob_checksum_on_device():
    rng = np.random.default_rng(8)
    x = np.maximum(rng.normal(0, 1, 4 << 20), 0).astype(np.float32)
    c, _ = pb.compress(pb.Tensor(x), pb.CodecParams(eb=1e-4))
    blob = c.to_bytes()
    assert len(blob) >= pc._DEVICE_CRC_MIN
    back = pc.CompressedActivation.from_bytes(blob)
    assert back.to_bytes() == blob
    bad = bytearray(blob)
    bad[len(bad) // 2] ^= 0x10
    with pytest.raises(FormatError, match="checksum"):
        pc.CompressedActivation.from_bytes(bytes(bad))
