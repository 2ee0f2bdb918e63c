"""Frequency-class codebook (k2r) parity: code lengths, canonical codes and
whole CMTZ blobs against the C oracle on activation-shaped histograms
(few frequency classes, wide alphabets, ties, class cuts), plus a check that
the fast path -- not the k2_codebook fallback -- produced them."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import _lib, huffman as ph  # noqa: E402


def _k2r_used() -> bool:
    L = _lib.lib()
    L.actc_debug_k2r_used.argtypes = [C.c_void_p]
    L.actc_debug_k2r_used.restype = C.c_int
    return bool(L.actc_debug_k2r_used(_lib.context().handle))


def _activation_hist(rng, A, n, width, kind):
    """Histogram of Lorenzo symbols of a ReLU-like activation: a spike at the
    zero delta plus a Laplace / Gaussian body of the given width."""
    r = A // 2
    if kind == "laplace":
        d = np.rint(rng.laplace(0, width, n)).astype(np.int64)
    else:
        d = np.rint(rng.normal(0, width, n)).astype(np.int64)
    d[rng.random(n) < 0.4] = 0
    d = d[np.abs(d) < r]
    return np.bincount(d + r, minlength=A).astype(np.uint64)


CASES = [
    ("laplace", 65536, 200_000, 30.0),
    ("laplace", 65536, 2_000_000, 300.0),
    ("laplace", 65536, 5_000_000, 3000.0),
    ("normal", 65536, 3_000_000, 9000.0),
    ("normal", 65536, 1_000_000, 20000.0),
    ("laplace", 4096, 1_000_000, 50.0),
    ("normal", 512, 100_000, 20.0),
]


@pytest.mark.parametrize("kind,A,n,width", CASES)
def test_code_lengths_activation_shaped(oracle, kind, A, n, width):
    rng = np.random.default_rng(int(width) + A)
    f = _activation_hist(rng, A, n, width, kind)
    got = ph.build_code_lengths(f)
    assert _k2r_used(), "frequency-class codebook did not run"
    assert np.array_equal(got, oracle.build_code_lengths(f))


def test_code_lengths_class_edge_cases(oracle):
    cases = []
    cases.append(np.ones(65536, dtype=np.uint64))                  # one class, all 16 bits
    cases.append(np.r_[np.ones(65535), [7]].astype(np.uint64))      # two classes
    x = np.zeros(65536, dtype=np.uint64)
    x[[3, 70000 % 65536]] = [5, 5]
    cases.append(x)                                                  # two equal live symbols
    x = np.zeros(300, dtype=np.uint64)
    x[17] = 9
    cases.append(x)                                                  # single live symbol
    fib = [1, 1]
    for _ in range(40):
        fib.append(fib[-1] + fib[-2])
    deep = np.array(fib, dtype=np.uint64)                           # 41 distinct lengths: fallback
    rng = np.random.default_rng(5)
    for A in (2, 3, 64, 1000, 65536):
        for hi in (2, 3, 50):
            cases.append(rng.integers(0, hi, A).astype(np.uint64))   # heavy ties
    for f in cases:
        got = ph.build_code_lengths(f)
        assert _k2r_used()
        assert np.array_equal(got, oracle.build_code_lengths(f))
    assert np.array_equal(ph.build_code_lengths(deep), oracle.build_code_lengths(deep))


def test_code_lengths_fallback_paths(oracle):
    rng = np.random.default_rng(9)
    # too many classes / weights over 2^32: k2_codebook runs and still matches
    f = rng.integers(1, 10 ** 6, 65536).astype(np.uint64)
    assert np.array_equal(ph.build_code_lengths(f), oracle.build_code_lengths(f))
    assert not _k2r_used()


@pytest.mark.parametrize("rel", [1e-3, 1e-4, 1e-5, 3e-6])
def test_codec_blob_tiny_eb_vs_oracle(oracle, rel):
    rng = np.random.default_rng(3)
    x = np.maximum(rng.normal(0, 1, (16, 64, 32, 32)), 0).astype(np.float32)
    x *= rng.random(x.shape[:2] + (1, 1)).astype(np.float32)
    eb = rel * float(x.max() - x.min())
    c, rep = pb.compress(pb.Tensor(x), pb.CodecParams(eb=eb))
    ref = oracle.compress(x, eb)
    assert c.to_bytes() == ref.blob
    assert rep.ratio == ref.ratio
    back = pb.decompress(c)
    want = oracle.decompress_blob(ref.blob, x.size)
    assert np.array_equal(back.data.view(np.uint64), want.view(np.uint64))
