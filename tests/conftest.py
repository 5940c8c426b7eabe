"""Test configuration.  `-m gpu` tests need a B200 (they call the CUDA path
through the C ABI); everything else runs on CPU.  The oracle (test
infrastructure under oracle/) and the golden vectors (tests/golden/) are
importable from here."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    import esn_oracle
    esn_oracle.build()
    return esn_oracle


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        return np.load(os.path.join(GOLDEN, f"ref_{name}.npz"))
    return load


@pytest.fixture(scope="session")
def esn():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1808_06736_b200 as E
    return E
