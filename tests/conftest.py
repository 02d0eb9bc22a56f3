import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLD = os.path.join(ROOT, "tests", "golden")
MODELS = os.path.join(GOLD, "models")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer statistical tests")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return dict(np.load(os.path.join(GOLD, "reference_golden.npz")))


@pytest.fixture(scope="session")
def models_dir():
    return MODELS


@pytest.fixture(scope="session")
def ref():
    """The reference library built from /root/reference (oracle/_ref); skipped when absent."""
    import reflib
    if not reflib.available():
        pytest.skip("oracle/_ref/libsst_ref.so not built (reference sources absent)")
    return reflib


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def renderer():
    """One B200 context for the session (fails loudly without a device)."""
    from paper_2011_03082_b200 import Renderer
    r = Renderer(0, "f32")
    r.load_models_dir(MODELS)
    yield r
    r.close()
