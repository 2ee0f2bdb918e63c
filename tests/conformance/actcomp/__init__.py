"""`actcomp` import shim for the conformance run: the reference's own unit
tests (pkg/tests/test_codec.py, test_huffman.py, unmodified) import
`actcomp.codec`, `actcomp.huffman`, `actcomp.tensor`, `actcomp.errors`; these
modules forward every hot-path name to the B200 drop-in
(paper_2111_09562_b200), so the tests exercise the CUDA path.  Test
infrastructure only; see run_reference_tests.sh."""
