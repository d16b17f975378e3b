import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: full-size configurations")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle, build
    build()
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Reference(False), Reference(True)


@pytest.fixture(scope="session")
def golden_small():
    return dict(np.load(os.path.join(GOLDEN, "small.npz")))


@pytest.fixture(scope="session")
def golden_hashes():
    with open(os.path.join(GOLDEN, "hashes.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gcoo():
    """The product package with its CUDA library (built if needed)."""
    from paper_2005_14469_b200 import build
    build.build()
    import paper_2005_14469_b200 as G
    G.lib()
    return G


@pytest.fixture(scope="session")
def cuda(gcoo):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    assert gcoo.device_count() >= 1, "libgcoo_cuda.so sees no device although torch does"
    return torch
