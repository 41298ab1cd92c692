"""Shared fixtures. `-m gpu` tests need a B200 and the built CUDA library;
`-m "not gpu"` tests run on CPU (oracle vs golden vectors, host logic, ABI
symbol checks, gloo multi-rank partitioning)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bind import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def known():
    with open(os.path.join(GOLDEN, "known_answers.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def refvec():
    with open(os.path.join(GOLDEN, "ref_vectors.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def reference():
    from oracle.bind import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()
