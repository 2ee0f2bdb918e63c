#!/bin/bash
# Run the reference's own hot-path unit tests, unmodified, against the B200
# drop-in through the `actcomp` shim.
#   stage (here, where /root/reference exists):  tests/conformance/run_reference_tests.sh stage
#   run   (GPU box, from the repo root):          tests/conformance/run_reference_tests.sh run
# The staged copies live in tests/conformance/_ref_tests/ (git-ignored: the
# reference's sources never enter the repository's history).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
case "$1" in
  stage)
    mkdir -p "$HERE/_ref_tests"
    cp /root/reference/pkg/tests/test_codec.py /root/reference/pkg/tests/test_huffman.py "$HERE/_ref_tests/"
    ;;
  run)
    ROOT=$(cd "$HERE/../.." && pwd)
    cd "$HERE/_ref_tests"
    PYTHONPATH="$HERE:$ROOT" python -m pytest -q -p no:cacheprovider --timeout 900 test_codec.py test_huffman.py
    ;;
  *) echo "usage: $0 stage|run"; exit 2 ;;
esac
