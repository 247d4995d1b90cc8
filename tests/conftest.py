import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a path")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle as O

    O.build()
    return O


@pytest.fixture(scope="session")
def gpu_ctx():
    """The product library (exact reference arithmetic)."""
    from paper_1408_2981_b200 import tpmg

    return tpmg.Context(device=0, variant="exact")


@pytest.fixture(scope="session")
def gpu_ctx_fma():
    """Experimental DFMA/reciprocal build (tolerance-level parity only)."""
    from paper_1408_2981_b200 import tpmg

    return tpmg.Context(device=0, variant="fma")


def rng_field(seed: int, n: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(n)
