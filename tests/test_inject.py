"""inject_uniform_error (reference errorprop.py:127-139): the oracle against
the reference's own outputs (tests/golden/make_inject_golden.py), and the
device kernel K7 bit-exact against both."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "inject_golden.npz")


def _cases():
    g = np.load(GOLDEN)
    i = 0
    while f"x_{i}" in g:
        eb, pz, seed = g[f"p_{i}"]
        yield g[f"x_{i}"], float(eb), bool(pz), int(seed), g[f"y_{i}"]
        i += 1


def test_oracle_matches_reference_golden(oracle):
    n = 0
    for x, eb, pz, seed, y in _cases():
        got = oracle.inject_uniform_error(x, eb, pz, seed)
        assert np.array_equal(got.view(np.uint64), y.reshape(-1).view(np.uint64))
        n += 1
    assert n == 5


@pytest.mark.gpu
def test_device_injection_bit_exact(oracle):
    torch = pytest.importorskip("torch")
    import paper_2111_09562_b200 as pb

    for x, eb, pz, seed, y in _cases():
        t = pb.Tensor(x, precision=4 if x.dtype == np.float32 else 8)
        got = pb.inject_uniform_error(t, eb, preserve_zeros=pz, seed=seed)
        assert got.precision == 8 and got.dims == x.shape
        assert np.array_equal(np.asarray(got.data).reshape(-1).view(np.uint64), y.reshape(-1).view(np.uint64))
    rng = np.random.default_rng(3)
    for n, dt, seed in ((3_000_001, np.float32, 11), (65_536 * 3 + 7, np.float64, 2 ** 62 + 1)):
        x = np.maximum(rng.normal(0, 1, n), 0).astype(dt)
        dev = pb.inject_uniform_error(torch.from_numpy(x).cuda(), 1e-2, seed=seed)
        assert dev.dtype == torch.float64 and dev.is_cuda
        want = oracle.inject_uniform_error(x, 1e-2, True, seed)
        assert np.array_equal(dev.cpu().numpy().view(np.uint64), want.view(np.uint64))
    with pytest.raises(pb.ParameterError):
        pb.inject_uniform_error(pb.Tensor(np.ones(4, np.float32)), 0.0)
