"""GPU conformance for the pipeline internals, mirroring the reference's
test_codec.py / test_huffman.py known answers and golden vectors."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200 import codec as pc, huffman as ph, tensor as pt  # noqa: E402
from paper_2111_09562_b200.errors import FormatError, ParameterError  # noqa: E402


def test_prequantize_known_answers(oracle):
    assert np.array_equal(pc.prequantize(np.array([0.0, 0.0, 0.0]), 1e-3), [0, 0, 0])
    assert pc.prequantize(np.array([0.0021]), 1e-3)[0] == 1
    assert pc.prequantize(np.array([0.003]), 1e-3)[0] == 2
    assert pc.prequantize(np.array([-0.003]), 1e-3)[0] == -2
    assert pc.prequantize(np.array([0.5 - 2.0 ** -54]), 0.5)[0] == 1
    with pytest.raises(ParameterError):
        pc.prequantize(np.array([1.0]), 0.0)
    rng = np.random.default_rng(0)
    for eb in (1e-2, 1e-3, 1e-4, 3e-7):
        x = rng.uniform(-5, 5, size=20000)
        assert np.array_equal(pc.prequantize(x, eb), oracle.prequantize(x, eb))
        x32 = x.astype(np.float32)
        assert np.array_equal(pc.prequantize(x32, eb), oracle.prequantize(x32, eb))


def test_lorenzo_known_answers():
    s, o = pc.lorenzo_encode(np.array([5, 5, 5, 5]), 100)
    assert list(s) == [105, 100, 100, 100] and len(o) == 0
    s, o = pc.lorenzo_encode(np.array([0, 10 ** 12]), 1 << 15)
    assert list(o) == [1] and s[1] == 0
    rng = np.random.default_rng(1)
    lat = rng.integers(-(10 ** 9), 10 ** 9, size=500)
    s, o = pc.lorenzo_encode(lat, 1 << 15)
    assert np.array_equal(pc.lorenzo_decode(s, lat[o], 1 << 15), lat)
    with pytest.raises(FormatError):
        s, o = pc.lorenzo_encode(np.array([0, 10 ** 12]), 1 << 15)
        pc.lorenzo_decode(s, [], 1 << 15)


def test_code_lengths_and_codes_golden(huffman_golden):
    j = 0
    while f"freq_{j}" in huffman_golden:
        f = huffman_golden[f"freq_{j}"]
        assert np.array_equal(ph.build_code_lengths(f), huffman_golden[f"len_{j}"]), j
        assert np.array_equal(ph.canonical_codes(huffman_golden[f"len_{j}"]), huffman_golden[f"codes_{j}"]), j
        j += 1


def test_code_lengths_random_vs_oracle(oracle):
    rng = np.random.default_rng(11)
    for trial in range(200):
        A = int(rng.choice([2, 3, 17, 256, 5000, 65536]))
        hi = int(rng.choice([2, 5, 100, 10 ** 6]))
        f = rng.integers(0, hi, size=A)
        if trial % 7 == 0:
            f[rng.integers(0, A)] = 10 ** 9
        assert np.array_equal(ph.build_code_lengths(f), oracle.build_code_lengths(f)), trial


def test_huffman_streams_golden(huffman_golden, golden_meta):
    for m in golden_meta["huffman"]:
        j = m["j"]
        s = huffman_golden[f"sym_{j}"]
        lengths, payload, bits = ph.huffman_encode(s, m["alphabet"])
        assert bits == m["bits"]
        assert np.array_equal(lengths, huffman_golden[f"symlen_{j}"])
        assert payload == huffman_golden[f"payload_{j}"].tobytes()
        assert np.array_equal(ph.huffman_decode(lengths, payload, bits, len(s)), s)


def test_huffman_reference_cases():
    syms = np.full(37, 5, dtype=np.int64)
    lengths, payload, bits = ph.huffman_encode(syms, 8)
    assert bits == 37 and lengths[5] == 1
    assert np.array_equal(ph.huffman_decode(lengths, payload, bits, 37), syms)
    lengths, payload, bits = ph.huffman_encode(np.array([0, 1, 0, 1]), 2)
    assert bits == 4 and list(lengths) == [1, 1]
    with pytest.raises(ParameterError):
        ph.huffman_encode(np.array([0, 9]), 4)
    syms = np.arange(16, dtype=np.int64)
    lengths, payload, bits = ph.huffman_encode(syms, 16)
    with pytest.raises(FormatError):
        ph.huffman_decode(lengths, payload[:1], bits, 16)
    with pytest.raises(FormatError):
        ph.huffman_decode(lengths, payload, bits // 2, 16)
    with pytest.raises(FormatError):
        ph.huffman_decode(np.zeros(8, dtype=np.uint16), b"\x00", 8, 3)
    rng = np.random.default_rng(5)
    syms = rng.integers(0, 65536, size=30000)
    lengths, payload, bits = ph.huffman_encode(syms, 65536)
    assert np.array_equal(ph.huffman_decode(lengths, payload, bits, len(syms)), syms)


def test_stats_vs_golden_and_oracle(stats_golden, golden_meta, oracle):
    s = golden_meta["stats"]
    act, grad, mom, mom64 = (stats_golden[k] for k in ("act", "grad", "mom", "mom64"))
    st = pt.compute_stats(act)
    assert st.nonzero_ratio == s["act_stats"]["nonzero_ratio"]
    assert st.mean_abs == s["act_stats"]["mean_abs"]
    assert st.max_abs == s["act_stats"]["max_abs"]
    per, lbar = pt.per_sample_max(torch.from_numpy(grad))
    assert list(per) == s["grad_per_sample_max"]
    assert lbar == s["grad_lbar_training"]
    assert pt.mean_abs(mom) == s["mom_mean_abs"]
    assert pt.mean_abs(mom64) == s["mom64_mean_abs"]
    ls = pb.collect_layer_stats("conv1", act, grad, mom, N=8)
    assert (ls.R, ls.L_bar, ls.M_avg) == (s["collect"]["R"], s["collect"]["L_bar"], s["collect"]["M_avg"])
    assert pb.plan_compression([ls], pb.ControllerConfig()).eb["conv1"] == s["plan_eb"]
    rng = np.random.default_rng(2)
    for n in (1, 7, 8, 129, 100003, 1 << 22, 25_000_017):
        a = rng.normal(size=n).astype(np.float32)
        assert pt.mean_abs(a) == float(np.abs(a).mean()), n
    g = rng.normal(size=(256, 4096)).astype(np.float32)
    _, lb = pt.per_sample_max(torch.from_numpy(g))
    assert lb == float(np.abs(g).reshape(256, -1).max(axis=1).mean())
