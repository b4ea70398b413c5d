import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: larger CPU oracle runs")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle_py import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from oracle.oracle_py import RefLib, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def golden_prims():
    return dict(np.load(os.path.join(GOLDEN, "primitives.npz")))


@pytest.fixture(scope="session")
def golden_ivf():
    return dict(np.load(os.path.join(GOLDEN, "ivf_small.npz")))


@pytest.fixture(scope="session")
def pq():
    """The product package (import fails loudly if the CUDA library is missing)."""
    import paper_1102_3828_b200 as p

    return p


@pytest.fixture(scope="session")
def golden_adc():
    return dict(np.load(os.path.join(GOLDEN, "adc_small.npz")))
