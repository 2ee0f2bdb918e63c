from paper_2111_09562_b200.codec import (CodecParams, CompressedActivation, CompressionReport,  # noqa: F401
                                         compress, decompress, lorenzo_decode, lorenzo_encode, prequantize,
                                         read_compressed, write_compressed)
