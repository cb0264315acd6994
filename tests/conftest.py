import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def ctx():
    """One product context for all GPU tests (n_max covers c5, the largest config)."""
    import torch
    import paper_0907_4631_b200 as P
    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but no CUDA device (the product has no CPU fallback)")
    P.build()
    c = P.Context(n_max=4_194_304, m_max=100, p_max=5)
    yield c
    c.close()
