import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
# the reference's own tests run against the drop-in through their own runner
# (tests/conformance/run_reference_tests.sh), not in the default suite
collect_ignore_glob = ["conformance/*"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")


@pytest.fixture(scope="session")
def golden_meta():
    with open(os.path.join(GOLDEN, "golden_meta.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def codec_golden():
    return np.load(os.path.join(GOLDEN, "codec_golden.npz"))


@pytest.fixture(scope="session")
def huffman_golden():
    return np.load(os.path.join(GOLDEN, "huffman_golden.npz"))


@pytest.fixture(scope="session")
def stats_golden():
    return np.load(os.path.join(GOLDEN, "stats_golden.npz"))


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc

    orc.build()
    return orc
