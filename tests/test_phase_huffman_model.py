"""CPU model of K2's phase-parallel two-queue Huffman merge.

K2 (csrc/k2_codebook.cu) claims: with leaves sorted by (freq, symbol) and
internal nodes kept in creation order, popping every item of frequency < 2m
(m = current minimum) in merged (freq, leaf-before-internal, index) order and
pairing consecutive items -- plus pairing an odd leftover with the smallest
remaining item -- reproduces heapq's pop order in build_code_lengths
(huffman.py:37-75).  This test runs that exact phase procedure in Python and
compares the resulting code lengths with the oracle (itself pinned to the
reference) on random, tie-heavy and Fibonacci frequency vectors.
"""
import numpy as np


def phase_lengths(freqs):
    freqs = np.asarray(freqs, dtype=np.int64)
    live = np.flatnonzero(freqs > 0)
    L = len(live)
    lengths = np.zeros(len(freqs), dtype=np.int64)
    if L == 0:
        return lengths
    if L == 1:
        lengths[live[0]] = 1
        return lengths
    order = sorted(range(L), key=lambda i: (freqs[live[i]], i))  # stable (freq, symbol)
    lf = [int(freqs[live[i]]) for i in order]
    nf, lpar, npar = [], [0] * L, []
    lp = np_ = 0
    phases = 0
    while (L - lp) + (len(nf) - np_) > 1:
        phases += 1
        m = min(lf[lp] if lp < L else 1 << 62, nf[np_] if np_ < len(nf) else 1 << 62)
        T = 2 * m
        na = sum(1 for i in range(lp, L) if lf[i] < T)
        nb = sum(1 for j in range(np_, len(nf)) if nf[j] < T)
        merged = []
        i = j = 0
        while i < na or j < nb:  # leaf wins ties
            if j >= nb or (i < na and lf[lp + i] <= nf[np_ + j]):
                merged.append(("L", lp + i, lf[lp + i]))
                i += 1
            else:
                merged.append(("N", np_ + j, nf[np_ + j]))
                j += 1
        tot = len(merged)
        nn = len(nf)
        for t in range(tot // 2):
            x, y = merged[2 * t], merged[2 * t + 1]
            nf.append(x[2] + y[2])
            npar.append(None)
            for it in (x, y):
                if it[0] == "L":
                    lpar[it[1]] = nn + t
                else:
                    npar[it[1]] = nn + t
        nlp, nnp = lp + na, np_ + nb
        if tot % 2:
            z = merged[-1]
            fl = lf[nlp] if nlp < L else 1 << 62
            fi = nf[nnp] if nnp < len(nf) else 1 << 62
            if nlp < L and fl <= fi:
                y = ("L", nlp, fl)
                nlp += 1
            else:
                y = ("N", nnp, fi)
                nnp += 1
            node = len(nf)
            nf.append(z[2] + y[2])
            npar.append(None)
            for it in (z, y):
                if it[0] == "L":
                    lpar[it[1]] = node
                else:
                    npar[it[1]] = node
        lp, np_ = nlp, nnp
    depth = [0] * len(nf)
    for k in range(len(nf) - 2, -1, -1):  # parents have larger indices
        depth[k] = depth[npar[k]] + 1
    for i in range(L):
        lengths[live[order[i]]] = depth[lpar[i]] + 1
    assert phases <= 64
    return lengths


def test_phase_model_matches_heapq_order(oracle):
    rng = np.random.default_rng(123)
    cases = []
    for _ in range(600):
        A = int(rng.integers(2, 300))
        kind = rng.integers(0, 4)
        if kind == 0:
            f = rng.integers(0, 50, size=A)
        elif kind == 1:
            f = rng.integers(0, 3, size=A)  # tie heavy
        elif kind == 2:
            f = (rng.pareto(1.2, size=A) * 10).astype(np.int64)
        else:
            f = rng.integers(0, 10 ** 6, size=A)
        cases.append(f)
    fib = [1, 1]
    while len(fib) < 40:
        fib.append(fib[-1] + fib[-2])
    cases += [np.array(fib[:30]), np.array(fib[:40][::-1]), np.ones(777, dtype=np.int64),
              np.array([1, 1, 2, 2, 4, 4, 8, 8, 16, 16, 32])]
    for f in cases:
        assert np.array_equal(phase_lengths(f), oracle.build_code_lengths(f).astype(np.int64)), f
