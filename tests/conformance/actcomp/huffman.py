"""Huffman entry points of the drop-in (GPU).  `_decode_tables` and
`_decode_bits_py` are reference internals one test calls directly
(huffman.py:97-142); they are restated here in plain Python as test
infrastructure (the drop-in decodes on the GPU)."""
import numpy as np

from paper_2111_09562_b200.huffman import (build_code_lengths, canonical_codes, huffman_decode,  # noqa: F401
                                           huffman_encode, stream_entropy_bits)


def _decode_tables(lengths):
    lengths = np.asarray(lengths, dtype=np.int64)
    max_len = int(lengths.max(initial=0))
    counts = np.bincount(lengths[lengths > 0], minlength=max_len + 1).astype(np.int64)[: max_len + 1]
    first = np.zeros(max_len + 1, dtype=np.int64)
    base = np.zeros(max_len + 1, dtype=np.int64)
    code = idx = 0
    for ln in range(1, max_len + 1):
        code <<= 1
        first[ln], base[ln] = code, idx
        code += counts[ln]
        idx += counts[ln]
    coded = np.flatnonzero(lengths > 0)
    order = coded[np.lexsort((coded, lengths[coded]))]
    return first, counts, base, order.astype(np.int64)


def _decode_bits_py(payload, bit_length, count, first, counts, base, syms, out):
    max_len = len(counts) - 1
    code = length = emitted = 0
    for pos in range(bit_length):
        code = (code << 1) | ((int(payload[pos >> 3]) >> (7 - (pos & 7))) & 1)
        length += 1
        if length > max_len:
            return -2
        off = code - int(first[length])
        if 0 <= off < int(counts[length]):
            out[emitted] = syms[int(base[length]) + off]
            emitted += 1
            if emitted == count:
                return pos + 1
            code = length = 0
    return -1
