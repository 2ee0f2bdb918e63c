"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports /root/reference/pkg/src/actcomp read-only (numba cache redirected
to /tmp, no bytecode written) and records, for a grid of adversarial inputs,
the exact CMTZ blob, report fields, the fp64 reconstruction, Huffman tables
and statistics.  The oracle (oracle/actc_oracle.c) is pinned against these
fixtures by tests/test_oracle_golden.py; the CUDA path is then checked
against the oracle (and directly against these fixtures) by the gpu tests.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

import actcomp  # noqa: E402
from actcomp import codec, huffman, controller, tensor  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def relu_normal(n, seed):
    return np.maximum(np.random.default_rng(seed).normal(0, 1, n), 0).astype(np.float32)


def rel_eb(x, rel):
    # the harness conversion used for "relative eb"
    return rel * float(x.max() - x.min()) if x.size else rel


def find_tie_outliers(eb, count, seed):
    """fp32 values whose reference bound check fails (fp64 ties)."""
    rng = np.random.default_rng(seed)
    found = []
    two = 2.0 * eb
    tries = 0
    while len(found) < count and tries < 2_000_000:
        k = int(rng.integers(0, 1 << 20))
        base = np.float32((k + 0.5) * two)
        cands = [base]
        c = base
        for _ in range(3):
            c = np.nextafter(c, np.float32(np.inf)); cands.append(c)
        c = base
        for _ in range(3):
            c = np.nextafter(c, np.float32(-np.inf)); cands.append(c)
        for v in cands:
            tries += 1
            vals = np.array([v], dtype=np.float64)
            q = codec.prequantize(vals, eb)
            rec = q.astype(np.float64) * two
            if np.abs(vals - rec)[0] > eb:
                found.append(np.float32(v))
    return np.array(found, dtype=np.float32)


def codec_cases():
    cases = []

    def add(name, x, eb, radius=codec.DEFAULT_RADIUS, preserve=True):
        cases.append((name, np.ascontiguousarray(x, dtype=np.float32), float(eb), int(radius), bool(preserve)))

    x = relu_normal(4096, 1)
    for rel in (1e-1, 1e-2, 1e-3, 1e-4):
        add(f"relu4096_rel{rel:g}", x, rel_eb(x, rel))
    x = relu_normal(20000, 2).reshape(5, 4, 1000)
    add("relu_rank3_rel1e-2_nopreserve", x, rel_eb(x, 1e-2), preserve=False)
    # config-1 shaped slice (same generator as C1, smaller batch)
    x = np.maximum(np.random.default_rng(0).normal(0, 1, 2 * 64 * 56 * 56), 0).astype(np.float32).reshape(2, 64, 56, 56)
    add("c1slice_rel1e-2", x, rel_eb(x, 1e-2))
    add("c1slice_rel1e-4", x, rel_eb(x, 1e-4))
    # reference make_tensor generator, relu-sparse (tensor.py:157-165)
    t = tensor.make_tensor([64, 100], "relu-sparse", sparsity=0.5, seed=0, precision=4)
    add("make_tensor_relu_sparse_eb0.01", t.view(), 0.01)
    t = tensor.make_tensor([3000], "uniform", lo=-1, hi=1, seed=5, precision=4)
    add("uniform3000_eb1e-3", t.view(), 1e-3)
    # ties that force outliers through the fp64 bound check
    for eb, seed in ((1e-3, 11), (0.053217172622680664, 12), (3e-5, 13)):
        ties = find_tie_outliers(eb, 16, seed)
        mix = np.concatenate([ties, relu_normal(200, seed), ties[::-1]])
        add(f"ties_eb{eb:g}", mix, eb)
    # exact binary half-integers (v = k + 0.5 exactly: no violation, q = k+1)
    eb = 2.0 ** -10
    k = np.arange(-50, 50)
    add("exact_halves_pow2eb", ((k + 0.5) * 2 * eb).astype(np.float32), eb)
    # floor(|v| + 0.5) rounding subtleties: v = 0.5 - 2^-54 and odd v in [2^52, 2^53)
    eb = 0.5
    add("rounding_edges", np.array([0.5 - 2.0 ** -25, 2.0 ** 24 - 1, 2.0 ** 23 + 1, -(2.0 ** 23 + 1), 3.0, -0.0, 0.0], dtype=np.float32), eb)
    eb = 2.0 ** -30
    add("rounding_edges_big_v", np.array([1.0, 3.0, 2.0 ** 22 + 1, -(2.0 ** 21 + 3), 7.0], dtype=np.float32), eb)
    # saturation: |v| >= 2^61 and inf
    add("saturation_inf", np.array([3e38, -3e38, 1.0, 0.0, 1e-30, -2.5], dtype=np.float32), 1e-300)
    add("saturation_2p61", np.array([1e10, -1e10, 2e10, 1.0], dtype=np.float32), 1e-9)
    # huge deltas / outliers
    add("outliers_huge", np.array([0.0, 1e9, 0.5, -1e9, 0.25, 0.0, 3.0], dtype=np.float32), 1e-3)
    add("rezero_outlier_path", np.array([1e9, 5e-4], dtype=np.float32), 1e-3)
    add("rezero_outlier_path_off", np.array([1e9, 5e-4], dtype=np.float32), 1e-3, preserve=False)
    # degenerate
    add("all_zero_10000", np.zeros(10000, np.float32), 1e-3)
    add("negzero", np.array([-0.0, -0.0, 0.0, -0.0], dtype=np.float32), 1e-3)
    add("constant_5000", np.full(5000, 0.25, np.float32), 1e-3)
    add("two_symbols", np.array([0.0, 1.0] * 50, dtype=np.float32), 0.25)
    for n in range(1, 9):
        add(f"tiny_n{n}", relu_normal(n, 100 + n) - 0.3, 1e-2)
    # fp32 subnormals
    add("subnormal", np.array([1e-45, 3e-44, -1e-40, 0.0, 1e-38], dtype=np.float32), 1e-46)
    # radius variants (u32 symbols beyond 2^16 alphabet)
    x = np.random.default_rng(7).uniform(-1, 1, 3000).astype(np.float32)
    for r in (2, 3, 100, 1 << 16, 1 << 17):
        add(f"radius{r}", x, 1e-4, radius=r)
    # wide alphabet: deltas spread over the whole +-2^15 window
    x = np.random.default_rng(9).uniform(-1, 1, 30000).astype(np.float32)
    add("wide_alphabet", x, 1.0 / 60000)
    # normal (signed) data
    x = np.random.default_rng(10).normal(0, 1, 5000).astype(np.float32)
    add("normal5000_eb1e-2", x, 1e-2)
    # runs longer than 65535 in the RLE table happen for huge radius
    add("radius_big_rle_split", np.array([0.1, 0.2, 0.1], dtype=np.float32), 1e-3, radius=1 << 18)
    return cases


def main():
    out = {}
    meta = []
    for i, (name, x, eb, radius, preserve) in enumerate(codec_cases()):
        t = tensor.Tensor(x)
        params = codec.CodecParams(eb=eb, radius=radius, preserve_zeros=preserve)
        c, rep = codec.compress(t, params)
        blob = c.to_bytes()
        back = codec.decompress(codec.CompressedActivation.from_bytes(blob))
        recon = back.data
        out[f"x_{i}"] = x
        out[f"blob_{i}"] = np.frombuffer(blob, dtype=np.uint8)
        keep_recon = x.size <= 20000
        if keep_recon:
            out[f"recon_{i}"] = recon
        meta.append(
            dict(
                i=i, name=name, dims=list(x.shape), eb=eb, radius=radius, preserve=preserve,
                n=int(x.size), k=int(len(c.outlier_indices)), payload_bits=int(c.payload_bits),
                compressed_bytes=rep.compressed_bytes, original_bytes=rep.original_bytes,
                ratio=rep.ratio, outlier_fraction=rep.outlier_fraction,
                entropy=rep.codes_entropy_bits_per_symbol, outlier_warning=rep.outlier_warning,
                recon_sha256=hashlib.sha256(np.ascontiguousarray(recon).tobytes()).hexdigest(),
                recon_stored=keep_recon,
            )
        )
        print(f"{i:3d} {name:34s} n={x.size:7d} k={meta[-1]['k']:4d} bytes={rep.compressed_bytes:8d} ratio={rep.ratio:.4f}")
    np.savez_compressed(os.path.join(HERE, "codec_golden.npz"), **out)

    # ---- Huffman-only vectors (huffman.py) ----
    hout = {}
    hmeta = []
    rng = np.random.default_rng(42)
    fib = [1, 1]
    while len(fib) < 40:
        fib.append(fib[-1] + fib[-2])
    freq_cases = [
        np.array([0, 10, 0, 0]), np.array([5, 5]), np.array([1000, 10, 10, 10]),
        np.array([3, 3, 3, 3, 1]), np.array([10, 7, 3, 1, 1, 20]), np.array([4, 4, 4, 4]),
        rng.integers(0, 1000, size=64), rng.integers(0, 3, size=200), rng.integers(0, 5, size=4096),
        np.array(fib[:30]), np.array(fib[:40][::-1]), np.ones(1000, dtype=np.int64),
        np.array([1, 1, 2, 2, 4, 4, 8, 8, 16, 16, 32]), rng.integers(1, 1 << 40, size=300),
    ]
    for j, f in enumerate(freq_cases):
        f = np.asarray(f, dtype=np.int64)
        hout[f"freq_{j}"] = f
        hout[f"len_{j}"] = huffman.build_code_lengths(f)
        hout[f"codes_{j}"] = huffman.canonical_codes(hout[f"len_{j}"])
    sym_cases = [
        (np.full(37, 5, dtype=np.int64), 8), (np.array([0, 1, 0, 1]), 2),
        (rng.integers(0, 65536, size=30000), 65536), (rng.integers(0, 20, size=5000), 20),
        (rng.choice(32, size=20000, p=rng.dirichlet(np.ones(32) * 0.2)), 32),
    ]
    for j, (s, a) in enumerate(sym_cases):
        lengths, payload, bits = huffman.huffman_encode(s, a)
        hout[f"sym_{j}"] = np.asarray(s, dtype=np.int64)
        hout[f"symlen_{j}"] = lengths
        hout[f"payload_{j}"] = np.frombuffer(payload, dtype=np.uint8)
        hmeta.append(dict(j=j, alphabet=a, bits=int(bits),
                          entropy=huffman.stream_entropy_bits(np.bincount(s, minlength=a))))
    np.savez_compressed(os.path.join(HERE, "huffman_golden.npz"), **hout)

    # ---- statistics + controller (tensor.py, training.py, controller.py) ----
    smeta = {}
    srng = np.random.default_rng(5)
    act = np.maximum(srng.normal(size=(8, 16, 12, 12)), 0).astype(np.float32)
    grad = srng.normal(size=(8, 16, 12, 12)).astype(np.float32) * 1e-3
    mom = srng.normal(size=(3000,)).astype(np.float32) * 1e-2
    mom64 = srng.normal(size=(4099,)) * 1e-2
    sout = {"act": act, "grad": grad, "mom": mom, "mom64": mom64}
    st = tensor.compute_stats(tensor.Tensor(act))
    smeta["act_stats"] = dict(nonzero_ratio=st.nonzero_ratio, mean_abs=st.mean_abs, max_abs=st.max_abs)
    smeta["grad_lbar_training"] = float(np.abs(grad).reshape(grad.shape[0], -1).max(axis=1).mean())
    gs = tensor.compute_stats(tensor.Tensor(grad), batch_dim=0)
    smeta["grad_per_sample_max"] = list(gs.per_sample_max_abs)
    smeta["mom_mean_abs"] = tensor.compute_stats(tensor.Tensor(mom)).mean_abs
    smeta["mom64_mean_abs"] = tensor.compute_stats(tensor.Tensor(mom64)).mean_abs
    ls = controller.collect_layer_stats("conv1", tensor.Tensor(act), tensor.Tensor(grad), tensor.Tensor(mom), N=8)
    smeta["collect"] = dict(R=ls.R, L_bar=ls.L_bar, M_avg=ls.M_avg)
    plan = controller.plan_compression([ls], controller.ControllerConfig())
    smeta["plan_eb"] = plan.eb.get("conv1")
    np.savez_compressed(os.path.join(HERE, "stats_golden.npz"), **sout)

    with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
        json.dump(
            dict(
                generator="tests/golden/make_golden.py",
                reference="/root/reference/pkg (actcomp %s)" % actcomp.__version__,
                numpy=np.__version__,
                numba=__import__("numba").__version__,
                codec=meta, huffman=hmeta, stats=smeta,
            ),
            fh, indent=1,
        )


if __name__ == "__main__":
    main()
