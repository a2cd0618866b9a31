import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libblws_cuda.so)")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def O():
    """The CPU oracle (test infrastructure only)."""
    from oracle import oracle

    return oracle


@pytest.fixture(scope="session")
def G():
    """The GPU product path (fails loudly without the extension / a GPU)."""
    import paper_1012_0365_b200 as pkg

    pkg.api.lib()
    return pkg


def principal_angle(u1, u2):
    """max principal angle via the sine (tests/oracles.hpp:83-88)."""
    resid = u2 - u1 @ (u1.T @ u2)
    s = np.linalg.svd(resid, compute_uv=False)
    return float(np.arcsin(min(1.0, s[0]))) if len(s) else 0.0
